import sys
import numpy as np
sys.path.insert(0, ".")
import oracle
import paper_2111_12055_b200 as gbx
o = oracle.Restatement()
dev = gbx.Device(0)
f, t = o.g1(17, 64)
p0 = o.policy_init(21)
for opt in ("sgd", "adam"):
    rc, pr, elr, _ = o.fit_variant(p0, f, t, 1e-3, 1, 64, 4, optimizer=opt, loss="td" if opt == "sgd" else "kl") if False else o.fit_variant(p0, f, t, 1e-3, 1, 64, 4, optimizer=opt)
    for mc in (1, 2):
        p, el = dev.fit(p0, f, t, 1e-3, 1, 64, 4, optimizer=opt, max_ctas=mc) if opt == "adam" else dev.fit(p0, f, np.stack([(f[:,8]>3).astype(float), f[:,9].astype(float)],1), 1e-3, 1, 64, 4, loss="td", max_ctas=mc)
        if opt == "sgd":
            rc, pr, elr, _ = o.fit_variant(p0, f, np.stack([(f[:,8]>3).astype(float), f[:,9].astype(float)],1), 1e-3, 1, 64, 4, loss="td")
        d = np.abs(p.astype(np.float64) - pr)
        print(opt, "max_ctas", mc, "max diff", d.max(), "n>1e-7", int((d > 1e-7).sum()), "idx", np.nonzero(d > 1e-7)[0][:8])
