"""ctypes binding for the fp64 CPU oracle (oracle/nsso.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package never
imports this module.  Argument marshalling only; all arithmetic is in nsso.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnsso.so")
SRC = [os.path.join(HERE, "nsso.c"), os.path.join(HERE, "nsso.h")]


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2, no fast-math) if it is missing or stale."""
    stale = not os.path.exists(LIB_PATH) or any(
        os.path.getmtime(s) > os.path.getmtime(LIB_PATH) for s in SRC)
    if force or stale:
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-o", tmp,
                               os.path.join(HERE, "nsso.c"), "-lm"])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


class Prior(C.Structure):
    _fields_ = [("kind", C.c_int32), ("d", C.c_int32),
                ("lo", C.POINTER(C.c_double)), ("hi", C.POINTER(C.c_double)),
                ("mean", C.POINTER(C.c_double)), ("sd", C.POINTER(C.c_double))]


class Energy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("d", C.c_int32), ("n_comp", C.c_int32),
                ("n_data", C.c_int64), ("d_in", C.c_int32),
                ("w", C.POINTER(C.c_double)), ("mu", C.POINTER(C.c_double)),
                ("sigma", C.POINTER(C.c_double)), ("prec", C.POINTER(C.c_double)),
                ("data_x", C.POINTER(C.c_double)), ("data_y", C.POINTER(C.c_double)),
                ("c", C.c_double), ("sigma_y", C.c_double), ("jitter", C.c_double)]


class Config(C.Structure):
    _fields_ = [("n_live", C.c_int64), ("k", C.c_int64), ("steps", C.c_int32),
                ("width_rule", C.c_int32), ("width", C.c_double), ("dir_norm", C.c_int32),
                ("max_stepout", C.c_int32), ("max_shrink", C.c_int32),
                ("quadrature", C.c_int32), ("metric_reg", C.c_double),
                ("term_log_ratio", C.c_double), ("n_volume_sims", C.c_int32),
                ("max_dead", C.c_int64), ("seed", C.c_uint64), ("update_all", C.c_int32),
                ("mutation", C.c_int32)]


class StepInfo(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("e_star", C.c_double), ("probes", C.c_int64),
                ("energy_evals", C.c_int64), ("expansions", C.c_int64), ("shrinks", C.c_int64),
                ("null_moves", C.c_int64), ("init_evals", C.c_int64),
                ("log_z_det", C.c_double), ("log_z_live", C.c_double),
                ("terminated", C.c_int32), ("finalised", C.c_int32)]

    def as_dict(self) -> Dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.POINTER
        vp = C.c_void_p
        L.nsso_init.argtypes = [P(Prior), P(Energy), P(Config), P(vp)]
        L.nsso_init_ex.argtypes = [P(Prior), P(Energy), P(Config), C.c_int, P(vp)]
        for name in ("nsso_step", "nsso_info"):
            getattr(L, name).argtypes = [vp, P(StepInfo)]
        L.nsso_run.argtypes = [vp, C.c_int64, P(StepInfo)]
        L.nsso_finalise.argtypes = [vp]
        L.nsso_evidence.argtypes = [vp, P(C.c_double), P(C.c_double)]
        L.nsso_evidence_reps.argtypes = [vp, P(C.c_double)]
        L.nsso_samples.argtypes = [vp, P(C.c_double), P(C.c_double), C.c_int64, P(C.c_int64)]
        L.nsso_smc_init.argtypes = [P(Prior), P(Energy), P(Config), C.c_double, P(vp)]
        L.nsso_smc_stage.argtypes = [vp]
        L.nsso_smc_state.argtypes = [vp, P(C.c_double), P(C.c_double), P(C.c_int64), P(C.c_int32)]
        L.nsso_smc_next_beta.argtypes = [P(C.c_double), C.c_int64, C.c_double, C.c_double, P(C.c_double)]
        L.nsso_rw_step.argtypes = [vp, P(C.c_double), C.c_double, C.c_double, C.c_uint32, C.c_uint32, C.c_uint32,
                                    P(C.c_double), P(C.c_double), P(C.c_int32)]
        L.nsso_posterior.argtypes = [vp, C.c_double, P(C.c_double), P(C.c_double), P(C.c_double),
                                     P(C.c_double), C.c_int64]
        L.nsso_resample.argtypes = [vp, C.c_double, C.c_int64, C.c_uint64, P(C.c_int64), P(C.c_double)]
        L.nsso_should_terminate.argtypes = [vp, P(C.c_int32)]
        L.nsso_destroy.argtypes = [vp]
        L.nsso_destroy.restype = None
        L.nsso_set_live.argtypes = [vp, P(C.c_double), P(C.c_double), C.c_int64]
        L.nsso_get_live.argtypes = [vp, P(C.c_double), P(C.c_double)]
        L.nsso_get_metric.argtypes = [vp, P(C.c_double), P(C.c_double)]
        L.nsso_set_chain_subset.argtypes = [vp, P(C.c_int32), C.c_int64]
        L.nsso_get_trace.argtypes = [vp, P(C.c_int32), P(C.c_int32), P(C.c_int32),
                                     P(C.c_uint8), P(C.c_double), P(C.c_double)]
        L.nsso_dead.argtypes = [vp, P(C.c_double), P(C.c_int32), P(C.c_double), P(C.c_int32),
                                P(C.c_double), C.c_int64, P(C.c_int64)]
        L.nsso_volume_reps.argtypes = [vp, P(C.c_double)]
        L.nsso_direction.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_uint32, P(C.c_double)]
        L.nsso_philox.argtypes = [P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
        L.nsso_philox.restype = None
        L.nsso_draw_u32.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                    C.c_uint32]
        L.nsso_draw_u32.restype = C.c_uint32
        L.nsso_draw_uniform.argtypes = L.nsso_draw_u32.argtypes
        L.nsso_draw_uniform.restype = C.c_double
        L.nsso_draw_normals.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.c_uint32, C.c_int32, P(C.c_double)]
        L.nsso_draw_normals.restype = None
        L.nsso_energy_at.argtypes = [vp, P(C.c_double)]
        L.nsso_energy_at.restype = C.c_double
        L.nsso_log_prior_at.argtypes = [vp, P(C.c_double)]
        L.nsso_log_prior_at.restype = C.c_double
        L.nsso_slice_step.argtypes = [vp, P(C.c_double), C.c_double, P(C.c_double), C.c_double,
                                      C.c_double, C.c_uint32, C.c_uint32, C.c_uint32,
                                      P(C.c_double), P(C.c_double), P(C.c_int32)]
        _lib = L
    return _lib


STATUS = {0: "OK", 1: "INVALID_ARG", 2: "PRIOR_SUPPORT", 3: "NAN", 7: "STATE", 8: "CAPACITY"}


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: nsso status {code} ({STATUS.get(code, '?')})")
        self.code = code


def _check(code: int, where: str):
    if code != 0:
        raise OracleError(code, where)


def _dp(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a) -> Optional[np.ndarray]:
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ---- unit hooks --------------------------------------------------------------
def smc_next_beta(E, beta_t: float, rho: float) -> float:
    e = _f64(E)
    out = C.c_double()
    _check(lib().nsso_smc_next_beta(_dp(e), e.size, float(beta_t), float(rho), C.byref(out)), "nsso_smc_next_beta")
    return out.value


def philox(ctr: Sequence[int], key: Sequence[int]):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().nsso_philox(c, k, o)
    return list(o)


def draw_u32(seed, it, gid, phase, sub, q) -> int:
    return lib().nsso_draw_u32(seed, it, gid, phase, sub, q)


def draw_uniform(seed, it, gid, phase, sub, q) -> float:
    return lib().nsso_draw_uniform(seed, it, gid, phase, sub, q)


def draw_normals(seed, it, gid, phase, sub, d) -> np.ndarray:
    z = np.zeros(d)
    lib().nsso_draw_normals(seed, it, gid, phase, sub, d, _dp(z))
    return z


class Oracle:
    """One oracle NSS run (nsso_ctx)."""

    def __init__(self, problem, cfg: Dict, draw_live: bool = True, smc_rho: Optional[float] = None):
        """smc_rho: build an F3 tempered SMC-SS context (nsso_smc_init) instead of NS."""
        self.problem = problem
        self.cfg = dict(cfg)
        d = problem.d
        self._keep = []

        def keep(a):
            a = _f64(a)
            if a is not None:
                self._keep.append(a)
            return a

        pr = Prior(kind=problem.prior_kind, d=d, lo=_dp(keep(problem.lo)), hi=_dp(keep(problem.hi)),
                   mean=_dp(keep(problem.mean)), sd=_dp(keep(problem.sd)))
        en = Energy(kind=problem.energy_kind, d=d, n_comp=problem.n_comp, n_data=problem.n_data,
                    d_in=problem.d_in, w=_dp(keep(problem.w)), mu=_dp(keep(problem.mu)),
                    sigma=_dp(keep(problem.sigma)), prec=_dp(keep(problem.prec)),
                    data_x=_dp(keep(problem.data_x)), data_y=_dp(keep(problem.data_y)),
                    c=problem.c, sigma_y=problem.sigma_y, jitter=problem.jitter)
        cf = Config(**self.cfg)
        h = C.c_void_p()
        if smc_rho is not None:
            _check(lib().nsso_smc_init(C.byref(pr), C.byref(en), C.byref(cf), float(smc_rho), C.byref(h)),
                   "nsso_smc_init")
        else:
            _check(lib().nsso_init_ex(C.byref(pr), C.byref(en), C.byref(cf), int(draw_live), C.byref(h)),
                   "nsso_init")
        self._h = h
        self.d = d
        self.n = self.cfg["n_live"]
        self.k = self.cfg["k"]
        self.p = self.cfg["steps"]
        self.R = self.cfg["n_volume_sims"]
        self.smc = smc_rho is not None

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().nsso_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- sampler ----
    def step(self) -> Dict:
        info = StepInfo()
        _check(lib().nsso_step(self._h, C.byref(info)), "nsso_step")
        return info.as_dict()

    def run(self, max_iters: int = 1 << 40) -> Dict:
        info = StepInfo()
        _check(lib().nsso_run(self._h, max_iters, C.byref(info)), "nsso_run")
        return info.as_dict()

    def finalise(self):
        _check(lib().nsso_finalise(self._h), "nsso_finalise")

    def info(self) -> Dict:
        info = StepInfo()
        _check(lib().nsso_info(self._h, C.byref(info)), "nsso_info")
        return info.as_dict()

    def should_terminate(self) -> bool:
        f = C.c_int32()
        _check(lib().nsso_should_terminate(self._h, C.byref(f)), "nsso_should_terminate")
        return bool(f.value)

    def evidence(self):
        lz, err = C.c_double(), C.c_double()
        _check(lib().nsso_evidence(self._h, C.byref(lz), C.byref(err)), "nsso_evidence")
        return lz.value, err.value

    def evidence_reps(self) -> np.ndarray:
        out = np.zeros(self.R + 1)
        _check(lib().nsso_evidence_reps(self._h, _dp(out)), "nsso_evidence_reps")
        return out

    def samples(self):
        n = C.c_int64()
        _check(lib().nsso_samples(self._h, None, None, 0, C.byref(n)), "nsso_samples")
        x = np.zeros((n.value, self.d))
        lw = np.zeros(n.value)
        _check(lib().nsso_samples(self._h, _dp(x), _dp(lw), n.value, C.byref(n)), "nsso_samples")
        return x, lw

    def posterior(self, beta: float = 1.0, weights: bool = False):
        """F2: (log Z(beta) mean, std over replicas, Kish ESS[, normalised log weights])."""
        lz, err, ess = C.c_double(), C.c_double(), C.c_double()
        lw = None
        if weights:
            n = C.c_int64()
            _check(lib().nsso_samples(self._h, None, None, 0, C.byref(n)), "nsso_samples")
            lw = np.zeros(n.value)
        _check(lib().nsso_posterior(self._h, float(beta), C.byref(lz), C.byref(err), C.byref(ess), _dp(lw),
                                    0 if lw is None else lw.size), "nsso_posterior")
        out = (lz.value, err.value, ess.value)
        return out + (lw,) if weights else out

    def resample(self, m: int, seed: int, beta: float = 1.0):
        """F2: m equal-weight draws: (dead indices, positions)."""
        idx = np.zeros(m, np.int64)
        x = np.zeros((m, self.d))
        _check(lib().nsso_resample(self._h, float(beta), int(m), int(seed),
                                   idx.ctypes.data_as(C.POINTER(C.c_int64)), _dp(x)), "nsso_resample")
        return idx, x

    def dead(self):
        n = C.c_int64()
        _check(lib().nsso_dead(self._h, None, None, None, None, None, 0, C.byref(n)), "nsso_dead")
        N = n.value
        e, b, x = np.zeros(N), np.zeros(N), np.zeros((N, self.d))
        nl, g = np.zeros(N, np.int32), np.zeros(N, np.int32)
        _check(lib().nsso_dead(self._h, _dp(e), nl.ctypes.data_as(C.POINTER(C.c_int32)), _dp(b),
                               g.ctypes.data_as(C.POINTER(C.c_int32)), _dp(x), N, C.byref(n)),
               "nsso_dead")
        return dict(e=e, n_live=nl, birth=b, gid=g, x=x)

    # ---- parity hooks ----
    def set_live(self, x: np.ndarray, e: np.ndarray, next_iteration: int):
        x = _f64(x).reshape(self.n, self.d)
        e = _f64(e).reshape(self.n)
        _check(lib().nsso_set_live(self._h, _dp(x), _dp(e), next_iteration), "nsso_set_live")

    def get_live(self):
        x = np.zeros((self.n, self.d))
        e = np.zeros(self.n)
        _check(lib().nsso_get_live(self._h, _dp(x), _dp(e)), "nsso_get_live")
        return x, e

    def volume_reps(self) -> np.ndarray:
        out = np.zeros(self.R + 1)
        _check(lib().nsso_volume_reps(self._h, _dp(out)), "nsso_volume_reps")
        return out

    def direction(self, it: int, gid: int, step: int) -> np.ndarray:
        v = np.zeros(self.d)
        _check(lib().nsso_direction(self._h, it, gid, step, _dp(v)), "nsso_direction")
        return v

    def metric(self):
        L = np.zeros((self.d, self.d))
        w = C.c_double()
        _check(lib().nsso_get_metric(self._h, _dp(L), C.byref(w)), "nsso_get_metric")
        return L, w.value

    def set_chain_subset(self, chains: Optional[Sequence[int]]):
        if chains is None:
            _check(lib().nsso_set_chain_subset(self._h, None, -1), "nsso_set_chain_subset")
            return
        a = np.ascontiguousarray(np.asarray(chains, dtype=np.int32))
        _check(lib().nsso_set_chain_subset(self._h, a.ctypes.data_as(C.POINTER(C.c_int32)),
                                           a.size), "nsso_set_chain_subset")

    def trace(self) -> Dict:
        k, p = self.k, max(self.p, 1)
        # chains per iteration (F4 update-all and F3 SMC stages: all n)
        nch = self.n if (self.cfg.get("update_all", 0) or self.smc) else k
        dead = np.zeros(k, np.int32)
        dest = np.zeros(nch, np.int32)
        par = np.zeros(nch, np.int32)
        counts = np.zeros((nch, p, 4), np.uint8)
        margin = np.zeros((nch, p))
        es = C.c_double()
        i32 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))
        _check(lib().nsso_get_trace(self._h, i32(dead), i32(dest), i32(par),
                                    counts.ctypes.data_as(C.POINTER(C.c_uint8)), _dp(margin),
                                    C.byref(es)), "nsso_get_trace")
        return dict(dead_gid=dead, dest_gid=dest, parent_gid=par, counts=counts,
                    min_margin=margin, e_star=es.value)

    # ---- unit hooks ----
    def energy(self, x) -> float:
        x = _f64(x)
        return lib().nsso_energy_at(self._h, _dp(x))

    def log_prior(self, x) -> float:
        x = _f64(x)
        return lib().nsso_log_prior_at(self._h, _dp(x))

    # ---- F3 tempered SMC-SS ----
    def smc_stage(self):
        _check(lib().nsso_smc_stage(self._h), "nsso_smc_stage")

    def smc_state(self):
        """(beta, log Z, stage, resampled parents of the last stage)."""
        b, lz, t = C.c_double(), C.c_double(), C.c_int64()
        par = np.zeros(self.n, np.int32)
        _check(lib().nsso_smc_state(self._h, C.byref(b), C.byref(lz), C.byref(t),
                                    par.ctypes.data_as(C.POINTER(C.c_int32))), "nsso_smc_state")
        return b.value, lz.value, t.value, par

    def smc_run(self, max_stages: int = 10_000):
        for _ in range(max_stages):
            if self.smc_state()[0] >= 1.0:
                break
            self.smc_stage()
        return self.smc_state()

    def rw_step(self, x0, e0: float, e_star: float, it: int, gid: int, step: int):
        """F1: one constrained random-walk proposal (nsso_rw_step)."""
        x0 = _f64(x0)
        xo = np.zeros(self.d)
        eo = C.c_double()
        cnt = (C.c_int32 * 4)()
        _check(lib().nsso_rw_step(self._h, _dp(x0), e0, e_star, it, gid, step, _dp(xo), C.byref(eo), cnt),
               "nsso_rw_step")
        return xo, eo.value, list(cnt)

    def slice_step(self, x0, e0: float, v, w: float, e_star: float, it: int, gid: int, step: int):
        x0, v = _f64(x0), _f64(v)
        xo = np.zeros(self.d)
        eo = C.c_double()
        cnt = (C.c_int32 * 4)()
        _check(lib().nsso_slice_step(self._h, _dp(x0), e0, _dp(v), w, e_star, it, gid, step,
                                     _dp(xo), C.byref(eo), cnt), "nsso_slice_step")
        return xo, eo.value, list(cnt)
