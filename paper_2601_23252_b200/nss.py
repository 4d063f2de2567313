"""Python binding of the B200 NSS library (include/nss.h, libnss.so).

Argument marshalling only: every step of the method runs in the CUDA kernels
behind the C ABI.  There is no CPU fallback -- importing this module on a
machine without the built library, or calling it without a GPU, raises.
PyTorch is used only for device selection and, in multi-GPU runs, to broadcast
the communicator id (torch.distributed); the library owns its device memory.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnss.so")

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "PRIOR_SUPPORT", 3: "NAN", 4: "CUDA", 5: "COMM", 6: "OOM",
          7: "STATE", 8: "CAPACITY", 9: "UNSUPPORTED"}


class NssError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str = ""):
        super().__init__(f"{where}: nss status {code} ({STATUS.get(code, '?')}) {msg}".strip())
        self.code = code


class nss_prior(C.Structure):
    _fields_ = [("kind", C.c_int32), ("d", C.c_int32),
                ("lo", C.POINTER(C.c_double)), ("hi", C.POINTER(C.c_double)),
                ("mean", C.POINTER(C.c_double)), ("sd", C.POINTER(C.c_double))]


class nss_energy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("d", C.c_int32), ("n_comp", C.c_int32),
                ("n_data", C.c_int64), ("d_in", C.c_int32),
                ("w", C.POINTER(C.c_double)), ("mu", C.POINTER(C.c_double)),
                ("sigma", C.POINTER(C.c_double)), ("prec", C.POINTER(C.c_double)),
                ("data_x", C.POINTER(C.c_double)), ("data_y", C.POINTER(C.c_double)),
                ("c", C.c_double), ("sigma_y", C.c_double), ("jitter", C.c_double)]


class nss_config(C.Structure):
    _fields_ = [("n_live", C.c_int64), ("k", C.c_int64), ("steps", C.c_int32),
                ("width_rule", C.c_int32), ("width", C.c_double), ("dir_norm", C.c_int32),
                ("max_stepout", C.c_int32), ("max_shrink", C.c_int32),
                ("quadrature", C.c_int32), ("metric_reg", C.c_double),
                ("term_log_ratio", C.c_double), ("n_volume_sims", C.c_int32),
                ("max_dead", C.c_int64), ("seed", C.c_uint64), ("update_all", C.c_int32),
                ("mutation", C.c_int32)]


class nss_dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("nccl_uid", C.POINTER(C.c_uint8)),
                ("cuda_stream", C.c_void_p)]


class nss_step_info(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("e_star", C.c_double), ("probes", C.c_int64),
                ("energy_evals", C.c_int64), ("expansions", C.c_int64), ("shrinks", C.c_int64),
                ("null_moves", C.c_int64), ("init_evals", C.c_int64),
                ("log_z_det", C.c_double), ("log_z_live", C.c_double),
                ("terminated", C.c_int32), ("finalised", C.c_int32)]

    def as_dict(self) -> Dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


EXPORTS = ["nss_get_unique_id", "nss_init", "nss_step", "nss_steps", "nss_run", "nss_finalise",
           "nss_evidence", "nss_evidence_reps", "nss_samples", "nss_info", "nss_sync", "nss_destroy",
           "nss_last_error", "nss_set_live", "nss_get_live", "nss_get_metric", "nss_get_trace",
           "nss_dead", "nss_volume_reps", "nss_set_kernel_timing", "nss_kernel_time",
           "nss_launch_count", "nss_set_hrss_engine", "nss_get_hrss_engine",
           "nss_phase_times", "nss_set_overlap", "nss_set_graph",
           "nss_debug_stamps", "nss_lr_energy_batch", "nss_gp_energy_batch", "nss_set_chain_range", "nss_posterior", "nss_resample", "nss_smc_init", "nss_smc_stage", "nss_smc_state", "nss_smc_run",
           "nss_group_init", "nss_group_step", "nss_group_gather_live"]

_lib = None


def lib():
    """Load libnss.so (built by __graft_entry__.build()); raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    P, vp = C.POINTER, C.c_void_p
    L.nss_get_unique_id.argtypes = [P(C.c_uint8)]
    L.nss_init.argtypes = [P(nss_prior), P(nss_energy), P(nss_config), P(nss_dist), P(vp)]
    L.nss_step.argtypes = [vp, P(nss_step_info)]
    L.nss_steps.argtypes = [vp, C.c_int64]
    L.nss_run.argtypes = [vp, C.c_int64, P(nss_step_info)]
    L.nss_finalise.argtypes = [vp]
    L.nss_evidence.argtypes = [vp, P(C.c_double), P(C.c_double)]
    L.nss_evidence_reps.argtypes = [vp, P(C.c_double)]
    L.nss_samples.argtypes = [vp, P(C.c_double), P(C.c_double), C.c_int64, P(C.c_int64)]
    L.nss_info.argtypes = [vp, P(nss_step_info)]
    L.nss_sync.argtypes = [vp]
    L.nss_destroy.argtypes = [vp]
    L.nss_last_error.argtypes = [vp]
    L.nss_last_error.restype = C.c_char_p
    L.nss_set_live.argtypes = [vp, P(C.c_float), P(C.c_float), C.c_int64]
    L.nss_get_live.argtypes = [vp, P(C.c_float), P(C.c_float)]
    L.nss_get_metric.argtypes = [vp, P(C.c_double), P(C.c_double)]
    L.nss_get_trace.argtypes = [vp, P(C.c_int32), P(C.c_int32), P(C.c_int32), P(C.c_uint8),
                                P(C.c_float)]
    L.nss_dead.argtypes = [vp, P(C.c_float), P(C.c_int32), P(C.c_float), P(C.c_int32),
                           P(C.c_float), C.c_int64, P(C.c_int64)]
    L.nss_volume_reps.argtypes = [vp, P(C.c_double)]
    L.nss_set_kernel_timing.argtypes = [vp, C.c_int32]
    L.nss_kernel_time.argtypes = [vp, P(C.c_double), P(C.c_int64)]
    L.nss_launch_count.argtypes = [vp, P(C.c_int64)]
    L.nss_set_hrss_engine.argtypes = [vp, C.c_int32]
    L.nss_get_hrss_engine.argtypes = [vp, P(C.c_int32)]
    L.nss_phase_times.argtypes = [vp, P(C.c_double), P(C.c_int64)]
    L.nss_set_overlap.argtypes = [vp, C.c_int32]
    L.nss_set_graph.argtypes = [vp, C.c_int32]
    L.nss_debug_stamps.argtypes = [vp, P(C.c_uint64)]
    L.nss_lr_energy_batch.argtypes = [P(C.c_double), P(C.c_double), C.c_int64, C.c_int32, P(C.c_double),
                                      C.c_int64, P(C.c_double)]
    L.nss_set_chain_range.argtypes = [vp, C.c_int32, C.c_int32]
    L.nss_smc_init.argtypes = [P(nss_prior), P(nss_energy), P(nss_config), C.c_double, P(nss_dist), P(vp)]
    L.nss_smc_stage.argtypes = [vp]
    L.nss_smc_state.argtypes = [vp, P(C.c_double), P(C.c_double), P(C.c_int64), P(C.c_int32)]
    L.nss_smc_run.argtypes = [vp, C.c_int64, P(C.c_double)]
    L.nss_posterior.argtypes = [vp, C.c_double, P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_double),
                                C.c_int64]
    L.nss_resample.argtypes = [vp, C.c_double, C.c_int64, C.c_uint64, P(C.c_int64), P(C.c_double)]
    L.nss_gp_energy_batch.argtypes = [P(C.c_double), P(C.c_double), C.c_int64, C.c_int32, C.c_double,
                                      P(C.c_double), C.c_int64, P(C.c_double)]
    L.nss_group_init.argtypes = [P(nss_prior), P(nss_energy), P(nss_config), C.c_int32, P(vp)]
    L.nss_group_step.argtypes = [P(vp), C.c_int32, C.c_int64]
    L.nss_group_gather_live.argtypes = [P(vp), C.c_int32]
    _lib = L
    return L


def _f64(a) -> Optional[np.ndarray]:
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _dp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _fp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_float))


def _ip(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int32))


def lr_energy_batch(data_x: np.ndarray, data_y: np.ndarray, theta: np.ndarray) -> np.ndarray:
    """Logistic-regression energies of the probe rows `theta` from the tcgen05
    kernel (include/nss.h nss_lr_energy_batch)."""
    X = _f64(data_x)
    y = _f64(data_y)
    th = np.ascontiguousarray(np.atleast_2d(np.asarray(theta, dtype=np.float64)))
    out = np.zeros(th.shape[0])
    st = lib().nss_lr_energy_batch(_dp(X), _dp(y), X.shape[0], X.shape[1], _dp(th), th.shape[0], _dp(out))
    if st != 0:
        raise NssError(st, "nss_lr_energy_batch")
    return out


def gp_energy_batch(data_x: np.ndarray, data_y: np.ndarray, jitter: float, phi: np.ndarray) -> np.ndarray:
    """fp64 GP marginal-likelihood energies of the hyperparameter rows `phi`
    from the batched-Cholesky kernel (include/nss.h nss_gp_energy_batch)."""
    X = _f64(np.atleast_2d(data_x))
    y = _f64(data_y)
    ph = np.ascontiguousarray(np.atleast_2d(np.asarray(phi, dtype=np.float64)))
    out = np.zeros(ph.shape[0])
    st = lib().nss_gp_energy_batch(_dp(X), _dp(y), X.shape[0], X.shape[1], float(jitter), _dp(ph), ph.shape[0],
                                   _dp(out))
    if st != 0:
        raise NssError(st, "nss_gp_energy_batch")
    return out


class Sampler:
    """One NSS run on one GPU (nss_ctx).  `problem` is a workloads.Problem and
    `cfg` a workloads.config() dict."""

    def __init__(self, problem, cfg: Dict, stream: Optional[int] = None, dist=None,
                 smc_rho: Optional[float] = None):
        """dist: None (one GPU) or (rank, world, nccl_uid bytes) -- see
        paper_2601_23252_b200.dist.sharded_sampler.  smc_rho: build an F3
        tempered SMC-SS context (nss_smc_init) instead of NS."""
        self.problem = problem
        self.cfg = dict(cfg)
        self._keep = []
        self._h = C.c_void_p()

        def keep(a):
            a = _f64(a)
            if a is not None:
                self._keep.append(a)
            return a

        d = problem.d
        pr = nss_prior(kind=problem.prior_kind, d=d, lo=_dp(keep(problem.lo)), hi=_dp(keep(problem.hi)),
                       mean=_dp(keep(problem.mean)), sd=_dp(keep(problem.sd)))
        en = nss_energy(kind=problem.energy_kind, d=d, n_comp=problem.n_comp, n_data=problem.n_data,
                        d_in=problem.d_in, w=_dp(keep(problem.w)), mu=_dp(keep(problem.mu)),
                        sigma=_dp(keep(problem.sigma)), prec=_dp(keep(problem.prec)),
                        data_x=_dp(keep(problem.data_x)), data_y=_dp(keep(problem.data_y)),
                        c=problem.c, sigma_y=problem.sigma_y, jitter=problem.jitter)
        cf = nss_config(**self.cfg)
        dd = None
        self.rank, self.world = 0, 1
        if stream is not None or dist is not None:
            uid = None
            if dist is not None:
                self.rank, self.world, raw = int(dist[0]), int(dist[1]), bytes(dist[2])
                if len(raw) != 128:
                    raise ValueError("nccl uid must be 128 bytes")
                uid = (C.c_uint8 * 128).from_buffer_copy(raw)
                self._keep.append(uid)
            dd = nss_dist(rank=self.rank, world=self.world,
                          nccl_uid=C.cast(uid, C.POINTER(C.c_uint8)) if uid is not None else None,
                          cuda_stream=C.c_void_p(stream) if stream is not None else None)
        if smc_rho is not None:
            st = lib().nss_smc_init(C.byref(pr), C.byref(en), C.byref(cf), float(smc_rho),
                                    C.byref(dd) if dd is not None else None, C.byref(self._h))
        else:
            st = lib().nss_init(C.byref(pr), C.byref(en), C.byref(cf),
                                C.byref(dd) if dd is not None else None, C.byref(self._h))
        if st != 0:
            raise NssError(st, "nss_init")
        self.d, self.n, self.k = d, self.cfg["n_live"], self.cfg["k"]
        self.p, self.R = self.cfg["steps"], self.cfg["n_volume_sims"]
        self.smc = smc_rho is not None

    @classmethod
    def _wrap(cls, problem, cfg: Dict, handle: C.c_void_p, rank: int, world: int, keep):
        """A Sampler around an existing context (nss_group_init members)."""
        self = cls.__new__(cls)
        self.problem, self.cfg, self._keep, self._h = problem, dict(cfg), keep, handle
        self.rank, self.world = rank, world
        self.d, self.n, self.k = problem.d, self.cfg["n_live"], self.cfg["k"]
        self.p, self.R = self.cfg["steps"], self.cfg["n_volume_sims"]
        self.smc = False
        return self

    def _check(self, st: int, where: str):
        if st != 0:
            msg = lib().nss_last_error(self._h) if self._h else b""
            raise NssError(st, where, (msg or b"").decode())

    # ---- F3 tempered SMC-SS ----
    def smc_stage(self):
        self._check(lib().nss_smc_stage(self._h), "nss_smc_stage")

    def smc_state(self):
        """(beta, log Z, stage, resampled parents of the last stage)."""
        b, lz, t = C.c_double(), C.c_double(), C.c_int64()
        par = np.zeros(self.n, np.int32)
        self._check(lib().nss_smc_state(self._h, C.byref(b), C.byref(lz), C.byref(t), _ip(par)), "nss_smc_state")
        return b.value, lz.value, t.value, par

    def smc_run(self, max_stages: int = 10_000):
        lz = C.c_double()
        self._check(lib().nss_smc_run(self._h, int(max_stages), C.byref(lz)), "nss_smc_run")
        return self.smc_state()

    def posterior(self, beta: float = 1.0, weights: bool = False):
        """F2: (log Z(beta) mean, std over replicas, Kish ESS[, normalised log weights])."""
        lz, err, ess = C.c_double(), C.c_double(), C.c_double()
        lw = None
        if weights:
            n = C.c_int64()
            self._check(lib().nss_samples(self._h, None, None, 0, C.byref(n)), "nss_samples")
            lw = np.zeros(n.value)
        self._check(lib().nss_posterior(self._h, float(beta), C.byref(lz), C.byref(err), C.byref(ess), _dp(lw),
                                        0 if lw is None else lw.size), "nss_posterior")
        out = (lz.value, err.value, ess.value)
        return out + (lw,) if weights else out

    def resample(self, m: int, seed: int, beta: float = 1.0):
        """F2: m equal-weight posterior draws: (dead-store indices, positions)."""
        idx = np.zeros(m, np.int64)
        x = np.zeros((m, self.d))
        self._check(lib().nss_resample(self._h, float(beta), int(m), int(seed),
                                       idx.ctypes.data_as(C.POINTER(C.c_int64)), _dp(x)), "nss_resample")
        return idx, x

    def set_chain_range(self, c0: int, c1: int):
        """Run only HRSS chains [c0, c1) (what one rank of a sharded run does)."""
        self._check(lib().nss_set_chain_range(self._h, int(c0), int(c1)), "nss_set_chain_range")

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().nss_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- sampler ----
    def step(self, sync: bool = True) -> Optional[Dict]:
        if not sync:
            self._check(lib().nss_step(self._h, None), "nss_step")
            return None
        info = nss_step_info()
        self._check(lib().nss_step(self._h, C.byref(info)), "nss_step")
        return info.as_dict()

    def steps(self, count: int):
        self._check(lib().nss_steps(self._h, count), "nss_steps")

    def run(self, max_iters: int = 1 << 40) -> Dict:
        info = nss_step_info()
        self._check(lib().nss_run(self._h, max_iters, C.byref(info)), "nss_run")
        return info.as_dict()

    def finalise(self):
        self._check(lib().nss_finalise(self._h), "nss_finalise")

    def sync(self):
        self._check(lib().nss_sync(self._h), "nss_sync")

    def info(self) -> Dict:
        info = nss_step_info()
        self._check(lib().nss_info(self._h, C.byref(info)), "nss_info")
        return info.as_dict()

    def evidence(self):
        lz, err = C.c_double(), C.c_double()
        self._check(lib().nss_evidence(self._h, C.byref(lz), C.byref(err)), "nss_evidence")
        return lz.value, err.value

    def evidence_reps(self) -> np.ndarray:
        out = np.zeros(self.R + 1)
        self._check(lib().nss_evidence_reps(self._h, _dp(out)), "nss_evidence_reps")
        return out

    def samples(self):
        n = C.c_int64()
        self._check(lib().nss_samples(self._h, None, None, 0, C.byref(n)), "nss_samples")
        x = np.zeros((n.value, self.d))
        lw = np.zeros(n.value)
        self._check(lib().nss_samples(self._h, _dp(x), _dp(lw), n.value, C.byref(n)), "nss_samples")
        return x, lw

    def dead(self) -> Dict:
        n = C.c_int64()
        self._check(lib().nss_dead(self._h, None, None, None, None, None, 0, C.byref(n)), "nss_dead")
        N = n.value
        e, b = np.zeros(N, np.float32), np.zeros(N, np.float32)
        x = np.zeros((N, self.d), np.float32)
        nl, g = np.zeros(N, np.int32), np.zeros(N, np.int32)
        self._check(lib().nss_dead(self._h, _fp(e), _ip(nl), _fp(b), _ip(g), _fp(x), N, C.byref(n)), "nss_dead")
        return dict(e=e, n_live=nl, birth=b, gid=g, x=x)

    # ---- parity hooks ----
    def set_live(self, x: np.ndarray, e: np.ndarray, next_iteration: int):
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float32).reshape(self.n, self.d))
        e = np.ascontiguousarray(np.asarray(e, dtype=np.float32).reshape(self.n))
        self._check(lib().nss_set_live(self._h, _fp(x), _fp(e), next_iteration), "nss_set_live")

    def get_live(self):
        x = np.zeros((self.n, self.d), np.float32)
        e = np.zeros(self.n, np.float32)
        self._check(lib().nss_get_live(self._h, _fp(x), _fp(e)), "nss_get_live")
        return x, e

    def metric(self):
        L = np.zeros((self.d, self.d))
        w = C.c_double()
        self._check(lib().nss_get_metric(self._h, _dp(L), C.byref(w)), "nss_get_metric")
        return L, w.value

    def trace(self) -> Dict:
        k, p = self.k, max(self.p, 1)
        # chains per iteration (F4 update-all and F3 SMC stages: all n)
        nch = self.n if (self.cfg.get("update_all", 0) or self.smc) else k
        dead = np.zeros(k, np.int32)
        dest, par = np.zeros(nch, np.int32), np.zeros(nch, np.int32)
        counts = np.zeros((nch, p, 4), np.uint8)
        es = C.c_float()
        self._check(lib().nss_get_trace(self._h, _ip(dead), _ip(dest), _ip(par),
                                        counts.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(es)),
                    "nss_get_trace")
        return dict(dead_gid=dead, dest_gid=dest, parent_gid=par, counts=counts, e_star=es.value)

    def volume_reps(self) -> np.ndarray:
        out = np.zeros(self.R + 1)
        self._check(lib().nss_volume_reps(self._h, _dp(out)), "nss_volume_reps")
        return out

    # ---- measurement ----
    def set_kernel_timing(self, on: bool):
        self._check(lib().nss_set_kernel_timing(self._h, 1 if on else 0), "nss_set_kernel_timing")

    def kernel_time(self):
        ms, n = C.c_double(), C.c_int64()
        self._check(lib().nss_kernel_time(self._h, C.byref(ms), C.byref(n)), "nss_kernel_time")
        return ms.value, n.value

    def set_engine(self, engine: str):
        """"auto", "warp", "lane" or "batch" (include/nss.h nss_hrss_engine)."""
        code = {"auto": 0, "warp": 1, "lane": 2, "batch": 3}[engine]
        self._check(lib().nss_set_hrss_engine(self._h, code), "nss_set_hrss_engine")

    def engine(self) -> str:
        e = C.c_int32()
        self._check(lib().nss_get_hrss_engine(self._h, C.byref(e)), "nss_get_hrss_engine")
        return {1: "warp", 2: "lane", 3: "batch"}[e.value]

    def phase_times(self) -> Dict:
        """Summed ms and launches per phase since timing was enabled."""
        ms = (C.c_double * 5)()
        n = (C.c_int64 * 5)()
        self._check(lib().nss_phase_times(self._h, ms, n), "nss_phase_times")
        names = ("hrss", "select", "evidence", "metric", "energy")
        return {nm: (ms[i], n[i]) for i, nm in enumerate(names)}

    def set_overlap(self, on: bool):
        self._check(lib().nss_set_overlap(self._h, 1 if on else 0), "nss_set_overlap")

    def set_graph(self, on: bool):
        self._check(lib().nss_set_graph(self._h, 1 if on else 0), "nss_set_graph")

    def debug_stamps(self) -> np.ndarray:
        out = np.zeros(16, np.uint64)
        self._check(lib().nss_debug_stamps(self._h, out.ctypes.data_as(C.POINTER(C.c_uint64))),
                    "nss_debug_stamps")
        return out

    def launch_count(self) -> int:
        n = C.c_int64()
        self._check(lib().nss_launch_count(self._h, C.byref(n)), "nss_launch_count")
        return n.value


def shard_ranges(n: int, world: int):
    """gid range [lo, hi) of every rank of a sharded run (include/nss.h):
    rank q owns segments q*8/world .. (q+1)*8/world - 1 of the 8 fixed gid
    segments [floor(s n / 8), floor((s + 1) n / 8))."""
    if world < 1 or 8 % world:
        raise ValueError("world must divide 8")
    per = 8 // world
    return [((q * per * n) // 8, ((q + 1) * per * n) // 8) for q in range(world)]


class Group:
    """The `world` ranks of one sharded run emulated in this process on one GPU
    (nss_group_init): members[q] is rank q (a Sampler)."""

    def __init__(self, problem, cfg: Dict, world: int):
        keep = []

        def kp(a):
            a = _f64(a)
            if a is not None:
                keep.append(a)
            return a

        d = problem.d
        pr = nss_prior(kind=problem.prior_kind, d=d, lo=_dp(kp(problem.lo)), hi=_dp(kp(problem.hi)),
                       mean=_dp(kp(problem.mean)), sd=_dp(kp(problem.sd)))
        en = nss_energy(kind=problem.energy_kind, d=d, n_comp=problem.n_comp, n_data=problem.n_data,
                        d_in=problem.d_in, w=_dp(kp(problem.w)), mu=_dp(kp(problem.mu)),
                        sigma=_dp(kp(problem.sigma)), prec=_dp(kp(problem.prec)),
                        data_x=_dp(kp(problem.data_x)), data_y=_dp(kp(problem.data_y)),
                        c=problem.c, sigma_y=problem.sigma_y, jitter=problem.jitter)
        cf = nss_config(**cfg)
        self.world = int(world)
        self._arr = (C.c_void_p * self.world)()
        st = lib().nss_group_init(C.byref(pr), C.byref(en), C.byref(cf), self.world, self._arr)
        if st != 0:
            raise NssError(st, "nss_group_init")
        self.members = [Sampler._wrap(problem, cfg, C.c_void_p(self._arr[q]), q, self.world, keep)
                        for q in range(self.world)]
        self.ranges = shard_ranges(cfg["n_live"], self.world)

    def steps(self, count: int):
        st = lib().nss_group_step(self._arr, self.world, int(count))
        if st != 0:
            raise NssError(st, "nss_group_step", (lib().nss_last_error(self._arr[0]) or b"").decode())

    def gather_live(self):
        st = lib().nss_group_gather_live(self._arr, self.world)
        if st != 0:
            raise NssError(st, "nss_group_gather_live")

    def owned_live(self):
        """The live set assembled from every rank's own rows."""
        parts = [m.get_live() for m in self.members]
        x = np.zeros_like(parts[0][0])
        e = np.zeros_like(parts[0][1])
        for (a, b), (xq, eq) in zip(self.ranges, parts):
            x[a:b], e[a:b] = xq[a:b], eq[a:b]
        return x, e

    def dead(self):
        """Dead store: replicated records, positions summed over the ranks
        (each rank holds the rows of the points it owned)."""
        ds = [m.dead() for m in self.members]
        out = dict(ds[0])
        out["x"] = np.sum([q["x"].astype(np.float64) for q in ds], axis=0).astype(np.float32)
        for q in ds[1:]:
            for key in ("e", "n_live", "gid", "birth"):
                if not np.array_equal(q[key], ds[0][key]):
                    raise AssertionError(f"dead store field {key} differs between ranks")
        return out

    def close(self):
        for m in self.members:
            m.close()
