"""Thin ctypes binding of libtdvp.so (include/tdvp.h).  Argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libtdvp.so; there is no
CPU fallback.  If the library is missing or has no GPU, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TDVP_LIB") or os.path.join(_HERE, "libtdvp.so")
_lib = None

TDVP_ERRORS = {-1: "bad argument", -2: "non-finite input", -3: "invalid partition", -4: "CUDA/NCCL failure",
               -5: "numerical failure", -6: "call order"}


def _check_cuda(dev):
    """Make `dev` the current CUDA device of this thread (the handle is created
    on the current device) through the CUDA runtime libtdvp links."""
    lib()  # libtdvp first: the CUDA runtime it links is the one resolved below
    rt = C.CDLL("libcudart.so.12") if _cudart[0] is None else _cudart[0]
    _cudart[0] = rt
    if rt.cudaSetDevice(int(dev)) != 0:
        raise TdvpError(-4, f"cudaSetDevice({dev}) failed")


_cudart = [None]


class TdvpError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libtdvp error {code} ({TDVP_ERRORS.get(code, '?')}): {msg}")
        self.code = code


class tdvp_params(C.Structure):
    _fields_ = [("eps", C.c_double), ("w_max", C.c_double), ("krylov_k", C.c_int), ("krylov_tol", C.c_double),
                ("multiplet_delta", C.c_double), ("timing", C.c_int), ("n_devices", C.c_int),
                ("device_ids", C.POINTER(C.c_int)), ("rebalance", C.c_double), ("u1", C.c_int)]


class tdvp_stats(C.Structure):
    _fields_ = [("w_step", C.c_double), ("w_total", C.c_double), ("trunc_active", C.c_int), ("n_pair", C.c_int),
                ("n_back", C.c_int), ("krylov_breakdowns", C.c_int), ("svd_sweeps_max", C.c_int),
                ("step_ms", C.c_double), ("heff2_ms", C.c_double), ("heff2_flop", C.c_double),
                ("heff2_calls", C.c_int), ("heff1_ms", C.c_double), ("heff1_flop", C.c_double),
                ("svd_ms", C.c_double), ("gemm_launches", C.c_longlong), ("kernel_launches", C.c_longlong),
                ("svd_jac_ms", C.c_double), ("svd_jac_flop", C.c_double), ("svd_sweeps_total", C.c_int),
                ("lanczos2_ms", C.c_double), ("lanczos1_ms", C.c_double),
                ("env_ms", C.c_double), ("heff2_ms_bin", C.c_double * 4), ("heff2_flop_bin", C.c_double * 4),
                ("lz_vec_bytes", C.c_double), ("rebalances", C.c_int), ("svd_bj_ms", C.c_double),
                ("svd_bj_flop", C.c_double), ("svd_bj_calls", C.c_int), ("lz_ms_bin", C.c_double * 4),
                ("lz_bytes_bin", C.c_double * 4), ("heff2_flop_exec", C.c_double), ("heff1_flop_exec", C.c_double)]

    def as_dict(self):
        out = {}
        for k, _ in self._fields_:
            v = getattr(self, k)
            out[k] = list(v) if isinstance(v, C.Array) else v
        return out


_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_PD = C.POINTER(_D)

_SIGS = {
    "tdvp_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "tdvp_set_params": (C.c_int, [C.c_void_p, C.POINTER(tdvp_params)]),
    "tdvp_get_params": (C.c_int, [C.c_void_p, C.POINTER(tdvp_params)]),
    "tdvp_set_mpo": (C.c_int, [C.c_void_p, _I, _PD]),
    "tdvp_set_mps": (C.c_int, [C.c_void_p, _I, _PD, _PD]),
    "tdvp_step": (C.c_int, [C.c_void_p, C.c_double, C.c_int]),
    "tdvp_step1": (C.c_int, [C.c_void_p, C.c_double, C.c_int]),
    "tdvp_step_hybrid": (C.c_int, [C.c_void_p, C.c_double, C.c_int, _I]),
    "tdvp_measure_sz": (C.c_int, [C.c_void_p, _D]),
    "tdvp_measure_energy": (C.c_int, [C.c_void_p, _D]),
    "tdvp_measure_norm": (C.c_int, [C.c_void_p, _D]),
    "tdvp_overlap": (C.c_int, [C.c_void_p, C.c_void_p, _D, _D]),
    "tdvp_infidelity": (C.c_int, [C.c_void_p, C.c_void_p, _D]),
    "tdvp_set_partition": (C.c_int, [C.c_void_p, C.c_int, _I]),
    "tdvp_partition_balanced": (C.c_int, [C.c_int, C.c_int, _I, _I, _I]),
    "tdvp_reorthonormalize": (C.c_int, [C.c_void_p]),
    "tdvp_get_stats": (C.c_int, [C.c_void_p, C.POINTER(tdvp_stats)]),
    "tdvp_get_chi": (C.c_int, [C.c_void_p, _I]),
    "tdvp_get_mps": (C.c_int, [C.c_void_p, _PD, _PD]),
    "tdvp_last_error": (C.c_char_p, [C.c_void_p]),
    "tdvp_destroy": (None, [C.c_void_p]),
    "tdvp_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "tdvp_comm_init": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_char_p]),
    "tdvp_plan": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _I, C.c_int]),
    "tdvp_plan1": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _I, C.c_int]),
    "tdvp_partition": (C.c_int, [C.c_int, C.c_int, _I, _I]),
    "tdvp_get_partition": (C.c_int, [C.c_void_p, _I, _I, _I]),
    "tdvp_dmrg": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _D]),
    "tdvp_apply_heff2": (C.c_int, [C.c_int] * 6 + [_D] * 6),
    "tdvp_apply_heff1": (C.c_int, [C.c_int] * 5 + [_D] * 5),
    "tdvp_env_left": (C.c_int, [C.c_int] * 5 + [_D] * 4),
    "tdvp_env_right": (C.c_int, [C.c_int] * 5 + [_D] * 4),
    "tdvp_expm_lanczos_dense": (C.c_int, [C.c_int, _D, _D, C.c_double, C.c_double, C.c_int, _D]),
    "tdvp_svd_split": (C.c_int, [C.c_int, C.c_int, _D, C.c_int, C.c_double, C.c_double, C.c_double, _I, _D, _D, _D,
                                 _D]),
    "tdvp_zgemm": (C.c_int, [C.c_int] * 5 + [_D] * 3),
    "tdvp_bench_heff2": (C.c_int, [C.c_int] * 4 + [_D, _D, C.c_int, _D, _D]),
    "tdvp_bench_svd": (C.c_int, [C.c_int, C.c_int, _D, C.c_int, _D, _I]),
}


def lib():
    """Load libtdvp.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python -m paper_1912_06127_b200.build`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _c(a):
    """contiguous complex128 array -> double pointer"""
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a, a.ctypes.data_as(_D)


def _check(rc, h=None):
    if rc != 0:
        msg = lib().tdvp_last_error(h).decode() if h else ""
        raise TdvpError(rc, msg)


class Tdvp:
    """Handle over one libtdvp context (one device, or one rank)."""

    def __init__(self, L, d, D_mpo, chi_max, devices=None):
        """devices: CUDA device ids for a multi-device handle (tdvp_params.n_devices /
        device_ids; the handle is created on devices[0], segment q of a p-segment
        step runs on devices[q * len(devices) // p])."""
        self.L, self.d = L, d
        self.devices = [int(x) for x in devices] if devices else []
        h = C.c_void_p()
        if self.devices:
            _check_cuda(self.devices[0])
        _check(lib().tdvp_create(L, d, D_mpo, chi_max, C.byref(h)))
        self.h = h
        self.set_params()

    def close(self):
        if getattr(self, "h", None):
            lib().tdvp_destroy(self.h)
            self.h = None

    __del__ = close

    def set_params(self, eps=1e-12, w_max=0.0, krylov_k=8, multiplet_delta=1e-6, timing=False, krylov_tol=0.0,
                   rebalance=0.0, u1=False):
        nd = len(self.devices)
        ids = (C.c_int * max(1, nd))(*(self.devices or [0]))
        p = tdvp_params(eps, w_max, krylov_k, krylov_tol, multiplet_delta, int(bool(timing)), nd if nd > 1 else 1,
                        ids, float(rebalance), int(bool(u1)))
        _check(lib().tdvp_set_params(self.h, C.byref(p)), self.h)

    def set_mpo(self, W):
        D = [1] + [w.shape[3] for w in W]
        Ws = [_c(w)[0] for w in W]
        arr = (_D * len(Ws))(*[w.ctypes.data_as(_D) for w in Ws])
        _check(lib().tdvp_set_mpo(self.h, (C.c_int * len(D))(*D), arr), self.h)

    def set_mps(self, psi, lam):
        chi = [1] + [p.shape[2] for p in psi[:-1]] + [1]
        P = [_c(p)[0] for p in psi]
        Lm = [np.ascontiguousarray(l, dtype=np.float64) for l in lam]
        pa = (_D * len(P))(*[p.ctypes.data_as(_D) for p in P])
        la = (_D * max(1, len(Lm)))(*[l.ctypes.data_as(_D) for l in Lm])
        _check(lib().tdvp_set_mps(self.h, (C.c_int * len(chi))(*chi), pa, la), self.h)

    def step(self, dt, n_segments=1):
        _check(lib().tdvp_step(self.h, float(dt), int(n_segments)), self.h)

    def step1(self, dt, n_segments=1):
        """One one-site TDVP step (tdvp_step1): serial 1TDVP, or p1TDVP with n_segments > 1."""
        _check(lib().tdvp_step1(self.h, float(dt), int(n_segments)), self.h)

    def step_hybrid(self, dt, n_segments=1):
        """One hybrid 2TDVP -> 1TDVP step (tdvp_step_hybrid); returns 1 or 2."""
        used = C.c_int()
        _check(lib().tdvp_step_hybrid(self.h, float(dt), int(n_segments), C.byref(used)), self.h)
        return used.value

    def measure_sz(self):
        out = np.zeros(self.L)
        _check(lib().tdvp_measure_sz(self.h, out.ctypes.data_as(_D)), self.h)
        return out

    def measure_energy(self):
        e = C.c_double()
        _check(lib().tdvp_measure_energy(self.h, C.byref(e)), self.h)
        return e.value

    def measure_norm(self):
        e = C.c_double()
        _check(lib().tdvp_measure_norm(self.h, C.byref(e)), self.h)
        return e.value

    def overlap(self, other):
        """<self|other> (tdvp_overlap)."""
        re, im = C.c_double(), C.c_double()
        _check(lib().tdvp_overlap(self.h, other.h, C.byref(re), C.byref(im)), self.h)
        return complex(re.value, im.value)

    def infidelity(self, other):
        """I = 1 - |<a|b>| / sqrt(<a|a><b|b>) (PAPER.md benchmark section; tdvp_infidelity)."""
        out = C.c_double()
        _check(lib().tdvp_infidelity(self.h, other.h, C.byref(out)), self.h)
        return out.value

    def reorthonormalize(self):
        """Exact re-gauging into inverse-canonical form (tdvp_reorthonormalize)."""
        _check(lib().tdvp_reorthonormalize(self.h), self.h)

    def set_partition(self, bounds):
        """Explicit segment bounds [(s, e)] for n_segments = len(bounds); None = uniform rule."""
        if not bounds:
            _check(lib().tdvp_set_partition(self.h, 0, None), self.h)
            return
        starts = (C.c_int * len(bounds))(*[int(s) for s, _ in bounds])
        _check(lib().tdvp_set_partition(self.h, len(bounds), starts), self.h)

    def dmrg(self, n_sweeps, restarts=4):
        """Two-site DMRG sweeps (tdvp_dmrg); returns the energy after every sweep."""
        out = np.zeros(max(1, n_sweeps))
        _check(lib().tdvp_dmrg(self.h, int(n_sweeps), int(restarts), out.ctypes.data_as(_D)), self.h)
        return out[:n_sweeps]

    def partition(self):
        """The segment bounds [(s, e)] the handle currently uses (tdvp_get_partition)."""
        n = C.c_int()
        _check(lib().tdvp_get_partition(self.h, C.byref(n), None, None), self.h)
        ss, ee = (C.c_int * max(1, n.value))(), (C.c_int * max(1, n.value))()
        _check(lib().tdvp_get_partition(self.h, C.byref(n), ss, ee), self.h)
        return [(ss[q], ee[q]) for q in range(n.value)]

    def maybe_reorthonormalize(self, tol):
        """Reorthonormalise when the norm error |<psi|psi> - 1| exceeds tol
        ("if the error in the norm grows unacceptably large");
        returns whether it did."""
        if abs(self.measure_norm() - 1.0) > tol:
            self.reorthonormalize()
            return True
        return False

    def stats(self):
        s = tdvp_stats()
        _check(lib().tdvp_get_stats(self.h, C.byref(s)), self.h)
        return s.as_dict()

    def chi(self):
        out = (C.c_int * (self.L + 1))()
        _check(lib().tdvp_get_chi(self.h, out), self.h)
        return list(out)

    def get_mps(self, out=None):
        """The current MPS (inverse-canonical Psi_j, Lambda_b).  out = (psi, lam):
        caller-owned C-contiguous arrays (e.g. pinned host memory) filled in
        place when their shapes match the current bond dimensions."""
        chi = self.chi()
        shp = [(chi[j], self.d, chi[j + 1]) for j in range(self.L)]
        if (out is not None and len(out[0]) == self.L and len(out[1]) == self.L - 1
                and all(o.shape == s and o.dtype == np.complex128 and o.flags.c_contiguous
                        for o, s in zip(out[0], shp))
                and all(o.shape == (chi[b + 1],) and o.dtype == np.float64 and o.flags.c_contiguous
                        for b, o in enumerate(out[1]))):
            psi, lam = out
        else:
            psi = [np.zeros(s, dtype=np.complex128) for s in shp]
            lam = [np.zeros(chi[b + 1]) for b in range(self.L - 1)]
        pa = (_D * self.L)(*[p.ctypes.data_as(_D) for p in psi])
        la = (_D * max(1, self.L - 1))(*[l.ctypes.data_as(_D) for l in lam])
        _check(lib().tdvp_get_mps(self.h, pa, la), self.h)
        return psi, lam

    def comm_init(self, rank, world, uid: bytes):
        _check(lib().tdvp_comm_init(self.h, rank, world, uid), self.h)


def balanced_partition(L, p, chi):
    """Contiguous partition minimising the largest segment cost (tdvp_partition_balanced)."""
    ch = (C.c_int * (L + 1))(*[int(x) for x in chi])
    s, e = (C.c_int * p)(), (C.c_int * p)()
    rc = lib().tdvp_partition_balanced(L, p, ch, s, e)
    if rc != 0:
        raise TdvpError(rc, f"tdvp_partition_balanced(L={L}, p={p})")
    return [(s[q], e[q]) for q in range(p)]


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().tdvp_nccl_unique_id(buf))
    return buf.raw


# ---------------------------------------------------------------- host-only
def plan(L, p, h, q, one_site=False):
    """Per-segment op list of tdvp_step (tdvp_plan) or of tdvp_step1 (tdvp_plan1)."""
    buf = (C.c_int * (4 * 8 * (L + 8)))()
    n = (lib().tdvp_plan1 if one_site else lib().tdvp_plan)(L, p, h, q, buf, 8 * (L + 8))
    if n < 0:
        raise TdvpError(n, f"tdvp_plan(L={L}, p={p})")
    return [tuple(buf[4 * i:4 * i + 4]) for i in range(n)]


def partition(L, p):
    s = (C.c_int * p)()
    e = (C.c_int * p)()
    _check(lib().tdvp_partition(L, p, s, e))
    return list(zip(list(s), list(e)))


# ------------------------------------------------------- kernel-level entries
def apply_heff2(Lenv, W1, W2, Renv, theta):
    cl, d, _, cr = theta.shape
    Dl, Dm, Dr = W1.shape[0], W1.shape[3], W2.shape[3]
    out = np.zeros_like(theta, dtype=np.complex128)
    args = [_c(x) for x in (Lenv, W1, W2, Renv, theta)]
    _check(lib().tdvp_apply_heff2(cl, cr, d, Dl, Dm, Dr, *[a[1] for a in args], out.ctypes.data_as(_D)))
    return out


def apply_heff1(Lenv, W, Renv, psi):
    cl, d, cr = psi.shape
    out = np.zeros_like(psi, dtype=np.complex128)
    args = [_c(x) for x in (Lenv, W, Renv, psi)]
    _check(lib().tdvp_apply_heff1(cl, cr, d, W.shape[0], W.shape[3], *[a[1] for a in args], out.ctypes.data_as(_D)))
    return out


def env_left(beta, A, W):
    cl, d, cr = A.shape
    out = np.zeros((cr, W.shape[3], cr), dtype=np.complex128)
    args = [_c(x) for x in (beta, A, W)]
    _check(lib().tdvp_env_left(cl, cr, d, W.shape[0], W.shape[3], *[a[1] for a in args], out.ctypes.data_as(_D)))
    return out


def env_right(gamma, B, W):
    cl, d, cr = B.shape
    out = np.zeros((cl, W.shape[0], cl), dtype=np.complex128)
    args = [_c(x) for x in (gamma, B, W)]
    _check(lib().tdvp_env_right(cl, cr, d, W.shape[0], W.shape[3], *[a[1] for a in args], out.ctypes.data_as(_D)))
    return out


def expm_lanczos_dense(H, v, tau, K=8):
    n = v.shape[0]
    out = np.zeros(n, dtype=np.complex128)
    (hH, pH), (hv, pv) = _c(H), _c(v)
    _check(lib().tdvp_expm_lanczos_dense(n, pH, pv, float(np.real(tau)), float(np.imag(tau)), K,
                                         out.ctypes.data_as(_D)))
    return out


def svd_split(M, chi_max, eps=1e-12, w_max=0.0, delta=1e-6):
    m, n = M.shape
    k = min(m, n)
    pl = np.zeros((m, k), dtype=np.complex128)
    pr = np.zeros((k, n), dtype=np.complex128)
    lam = np.zeros(k)
    chi = C.c_int()
    w = C.c_double()
    hM, pM = _c(M)
    _check(lib().tdvp_svd_split(m, n, pM, chi_max, eps, w_max, delta, C.byref(chi), C.byref(w),
                                pl.ctypes.data_as(_D), lam.ctypes.data_as(_D), pr.ctypes.data_as(_D)))
    c = chi.value
    # psiL was written with row stride chi
    pl = pl.reshape(-1)[: m * c].reshape(m, c)
    pr = pr.reshape(-1)[: c * n].reshape(c, n)
    return pl, lam[:c], pr, w.value


def zgemm(opA, opB, A, B):
    ops = {"N": 0, "T": 1, "C": 2, "R": 3}
    a, b = ops[opA], ops[opB]
    M = A.shape[1] if a in (1, 2) else A.shape[0]
    K = A.shape[0] if a in (1, 2) else A.shape[1]
    N = B.shape[0] if b in (1, 2) else B.shape[1]
    out = np.zeros((M, N), dtype=np.complex128)
    (hA, pA), (hB, pB) = _c(A), _c(B)
    _check(lib().tdvp_zgemm(a, b, M, N, K, pA, pB, out.ctypes.data_as(_D)))
    return out


# ---------------------------------------------------------------- microbench
def bench_heff2(chi, W1, W2, reps=20):
    ms, fl = C.c_double(), C.c_double()
    (h1, p1), (h2, p2) = _c(W1), _c(W2)
    _check(lib().tdvp_bench_heff2(chi, W1.shape[0], W1.shape[3], W2.shape[3], p1, p2, reps, C.byref(ms), C.byref(fl)))
    return ms.value, fl.value


def bench_svd(M, reps=5):
    ms, sw = C.c_double(), C.c_int()
    hM, pM = _c(M)
    _check(lib().tdvp_bench_svd(M.shape[0], M.shape[1], pM, reps, C.byref(ms), C.byref(sw)))
    return ms.value, sw.value
