"""Small driver for ncu captures of the train / shuffle kernels."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2111_12055_b200 as gbx
from bench import synthetic_log

n = int(sys.argv[1]); batch = int(sys.argv[2])
feat, tgt = synthetic_log(n)
dev = gbx.Device(0)
p = dev.policy_init(7)
for _ in range(2):
    dev.fit(p, feat, tgt, 0.01, 1, batch, 99)
