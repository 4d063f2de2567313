"""Time the tcgen05 logistic-regression energy pass alone (kernel check path,
NSS_LR_REPS repeats timed with events inside the library) on the C4 data."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8000
if len(sys.argv) > 2:  # a variant library (scripts/build_lr_variants.sh)
    nss.LIB_PATH = os.path.abspath(sys.argv[2])
prob = W.logreg(100, 10_000)
theta = np.random.default_rng(1).standard_normal((P, 100)) * 0.3
os.environ.setdefault("NSS_LR_REPS", "50")
nss.lr_energy_batch(prob.data_x, prob.data_y, theta)
