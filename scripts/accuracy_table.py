"""Full NSS runs on the GPU at the BASELINE sizes against the analytic log Z
(north_star: |log Z - analytic| <= max(3 sigma_NS, 0.05)): C1 (Gaussian in a
box, erf form), C2 (4-component MoG in a box, erf products), C3a (correlated
Gaussian likelihood under a Gaussian prior, Gaussian convolution).  Writes a
markdown table to stdout."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from scipy import stats  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402


def truth_c1():
    return 2 * math.log(math.erf(5 / math.sqrt(2))) - 2 * math.log(10)


def truth_mog(prob):
    mass = [prob.w[j] * np.prod(stats.norm(prob.mu[j], prob.sigma[j]).cdf(prob.hi) -
                                stats.norm(prob.mu[j], prob.sigma[j]).cdf(prob.lo)) for j in range(len(prob.w))]
    return math.log(sum(mass)) - float(np.sum(np.log(prob.hi - prob.lo)))


def truth_corr(prob):
    # exp(-E) = exp(-c) exp(-1/2 (x-mu)^T P (x-mu)) = exp(-c) (2 pi)^{d/2} |P|^{-1/2} N(x; mu, P^-1);
    # Z = int N(x; 0, S0) exp(-E) dx = exp(-c) (2 pi)^{d/2} |P|^{-1/2} N(mu; 0, S0 + P^-1)
    d = prob.d
    P = np.asarray(prob.prec, dtype=np.float64)
    S0 = np.diag(np.asarray(prob.sd, dtype=np.float64) ** 2)
    _, logdetP = np.linalg.slogdet(P)
    cov = S0 + np.linalg.inv(P)
    lz = stats.multivariate_normal(mean=np.zeros(d), cov=cov).logpdf(np.asarray(prob.mu) - np.asarray(prob.mean))
    return -float(prob.c) + 0.5 * d * math.log(2 * math.pi) - 0.5 * logdetP + lz


def truth_funnel(prob):
    # box [-20, 20]^d (R-23): Z = |box|^-1 int_{-20}^{20} N(y; 0, sy^2) prod_{n<d} P(|x_n| <= 20 ; sd e^{y/2}) dy
    from scipy import integrate, special
    d, sy = prob.d, float(prob.sigma_y)
    half = float(prob.hi[0])

    def integrand(y):
        m = special.erf(half / (math.exp(y / 2) * math.sqrt(2)))
        return math.exp(stats.norm(0, sy).logpdf(y) + (d - 1) * math.log(max(m, 1e-300)))

    val, _ = integrate.quad(integrand, -half, half, points=[-10, -5, 0, 5], limit=400)
    return math.log(val) - d * math.log(2 * half)


def runs(name, prob, cfg, seeds):
    rows = []
    for s in seeds:
        g = nss.Sampler(prob, dict(cfg, seed=s))
        t0 = time.perf_counter()
        info = g.run()
        lz, sig = g.evidence()
        dt = time.perf_counter() - t0
        g.close()
        rows.append((s, lz, sig, info["iteration"], info["energy_evals"], dt))
    return rows


def main():
    big = 10_000 + 1000 * 8000  # a full d = 100 run takes several thousand iterations: dead store for 8000
    cases = [
        ("C1 gauss2", W.gauss(2), W.workload("C1")[1], truth_c1(), range(1, 9)),
        ("C2 mog10", W.mog(10), W.workload("C2")[1], None, range(1, 6)),
        # the BASELINE C3 settings: p = 3d HRSS steps, the paper's setting for
        # high-dimensional problems (R-35)
        ("C3a corrgauss100", W.workload("C3a")[0], dict(W.workload("C3a")[1], max_dead=big), None, range(1, 6)),
        ("C3b funnel100", W.workload("C3b")[0], dict(W.workload("C3b")[1], max_dead=big), None, range(1, 6)),
        # p = d, the round-1 setting, for comparison (the known bias at p = d, R-35)
        ("C3a corrgauss100 p=d", W.workload("C3a")[0], dict(W.workload("C3a")[1], max_dead=big, steps=100), None,
         range(1, 4)),
        ("C3b funnel100 p=d", W.workload("C3b")[0], dict(W.workload("C3b")[1], max_dead=big, steps=100), None,
         range(1, 4)),
    ]
    only = sys.argv[1:]  # optional case-name prefixes
    if only:
        cases = [c for c in cases if any(c[0].startswith(o) for o in only)]
    print("| config | seed | log Z | sigma_NS | analytic | abs diff | bound max(3 sigma, 0.05) | ok | iterations "
          "| energy evals | wall s (run() incl. finalise) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for name, prob, cfg, truth, seeds in cases:
        if truth is None:
            truth = (truth_mog(prob) if prob.energy_kind == W.E_MOG else
                     truth_funnel(prob) if prob.energy_kind == W.E_FUNNEL else truth_corr(prob))
        for s, lz, sig, it, ev, dt in runs(name, prob, cfg, seeds):
            diff = abs(lz - truth)
            bound = max(3 * sig, 0.05)
            print(f"| {name} | {s} | {lz:.4f} | {sig:.4f} | {truth:.4f} | {diff:.4f} | {bound:.4f} | "
                  f"{'yes' if diff <= bound else 'NO'} | {it} | {ev} | {dt:.2f} |", flush=True)


if __name__ == "__main__":
    main()
