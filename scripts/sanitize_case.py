"""A short workload for compute-sanitizer (tests/test_gpu_sanitizer.py): C1
and C2 iterations on the lane and warp engines, a batch-engine logistic
regression and GP, a sharded rank group, finalisation, evidence, posterior
samples.  Sizes are small: the sanitizer slows kernels 10-100x."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402


def main():
    cases = [(W.gauss(2), dict(n_live=200, k=20, steps=10), "auto"),
             (W.mog(10), dict(n_live=2000, k=200, steps=10), "auto"),
             (W.mog(10), dict(n_live=500, k=50, steps=4), "warp"),
             (W.logreg(5, n_data=300, seed=3), dict(n_live=256, k=32, steps=2), "auto"),
             (W.gp_ard(2, 40, seed=3), dict(n_live=64, k=16, steps=2), "auto")]
    for prob, kw, engine in cases:
        s = nss.Sampler(prob, W.config(seed=3, **kw))
        s.set_engine(engine)
        s.steps(3)
        s.step()
        s.finalise()
        s.evidence()
        s.samples()
        s.close()
    g = nss.Group(W.mog(10), W.config(seed=3, n_live=2000, k=200, steps=4), 4)
    g.steps(3)
    g.gather_live()
    for m in g.members:
        m.finalise()
        m.evidence()
    g.close()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
