"""Small driver for ncu captures of the inference kernels."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2111_12055_b200 as gbx
from bench import synthetic_log

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
feat, _ = synthetic_log(n)
dev = gbx.Device(0)
p = dev.policy_init(7)
for _ in range(2):
    dev.forward(p, feat, gbx.FWD_FAST)
