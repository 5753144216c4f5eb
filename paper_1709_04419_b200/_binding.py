"""Thin ctypes binding of include/hmlik.h (argument marshalling only).

Every computation runs inside libhmlik.so (CUDA kernels for sm_100a and the
host C++ runtime).  If the library is missing the import fails loudly; there
is no Python or CPU fallback for any entry point.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libhmlik.so")

HM_OK = 0
ERRORS = {-1: "HM_ERR_ARG", -2: "HM_ERR_CUDA", -3: "HM_ERR_NOT_SPD", -4: "HM_ERR_RANK_CAP",
          -5: "HM_ERR_OOM", -6: "HM_ERR_STATE", -7: "HM_ERR_TOO_LARGE"}


class HMError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class Theta(C.Structure):
    _fields_ = [("sigma2", C.c_double), ("ell", C.c_double), ("nu", C.c_double)]


class Params(C.Structure):
    _fields_ = [("eps", C.c_double), ("leaf", C.c_int32), ("eta", C.c_double), ("kmax", C.c_int32),
                ("rel_eps", C.c_int32), ("coop_max", C.c_int32), ("eps_chol", C.c_double),
                ("exec_ctas", C.c_int32), ("adaptive_cap", C.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found -- run `python -m paper_1709_04419_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "hm_last_error": ([], C.c_char_p),
        "hm_version": ([], C.c_char_p),
        "hm_tree_build": ([P, I64, I32, D, C.POINTER(P)], C.c_int),
        "hm_tree_free": ([P], C.c_int),
        "hm_tree_counts": ([P, P], C.c_int),
        "hm_tree_perm": ([P, P], C.c_int),
        "hm_tree_clusters": ([P, P], C.c_int),
        "hm_tree_blocks": ([P, P], C.c_int),
        "hm_plan_dump": ([P, I32, C.c_char_p, P], C.c_int),
        "hm_build": ([P, I32, I64, Theta, Params, I32, P, C.POINTER(P)], C.c_int),
        "hm_free": ([P], C.c_int),
        "hm_assemble": ([P, Theta], C.c_int),
        "hm_cholesky": ([P], C.c_int),
        "hm_loglik": ([P, P, I32, I32, P], C.c_int),
        "hm_loglik_batch": ([P, P, I32, P, I32, I32, P], C.c_int),
        "hm_sample": ([P, P, I32, I32, P, I32], C.c_int),
        "hm_stats": ([P, P], C.c_int),
        "hm_timings": ([P, P], C.c_int),
        "hm_profile": ([P, I32], C.c_int),
        "hm_kernel_stats": ([P, P], C.c_int),
        "hm_set_exec_mode": ([P, I32], C.c_int),
        "hm_set_exec_grid": ([P, I32], C.c_int),
        "hm_trace": ([P, I32, C.c_char_p], C.c_int),
        "hm_checksum": ([P, P], C.c_int),
        "hm_to_dense": ([P, P], C.c_int),
        "hm_loglik_multi": ([I32, P, P, P, I32, I32, P], C.c_int),
        "hm_set_batch_streams": ([P, I32], C.c_int),
        "hm_dense_loglik": ([P, I32, I64, Theta, P, I32, I32, I32, P, P], C.c_int),
        "hm_matern_block": ([P, I64, P, I64, Theta, I32, P], C.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


lib = _load()
EXPORTED = ("hm_last_error", "hm_version", "hm_tree_build", "hm_tree_free", "hm_tree_counts", "hm_tree_perm",
            "hm_tree_clusters", "hm_tree_blocks", "hm_plan_dump", "hm_build", "hm_free", "hm_assemble", "hm_cholesky",
            "hm_loglik", "hm_loglik_batch", "hm_sample", "hm_stats", "hm_timings", "hm_profile",
            "hm_kernel_stats", "hm_set_exec_mode", "hm_set_exec_grid", "hm_trace", "hm_checksum", "hm_to_dense", "hm_loglik_multi", "hm_set_batch_streams",
            "hm_dense_loglik", "hm_matern_block")


def check(code: int):
    if code != HM_OK:
        raise HMError(code, lib.hm_last_error().decode())


def _as_f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def ptr_of(a):
    """(pointer, on_device) for a numpy array or a torch tensor."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(C.c_void_p), 0
    import torch  # plumbing only: device memory + streams
    if isinstance(a, torch.Tensor):
        if a.dtype != torch.float64 or not a.is_contiguous():
            raise TypeError("tensor must be contiguous float64")
        return C.c_void_p(a.data_ptr()), 1 if a.is_cuda else 0
    raise TypeError(type(a))


# ---------------------------------------------------------------- geometry
class Tree:
    """Cluster tree + block cluster tree built by hm_tree_build (host C++)."""

    def __init__(self, locs, leaf: int, eta: float):
        locs = _as_f64(locs)
        if locs.ndim != 2 or locs.shape[1] != 2:
            raise ValueError("locs must be n x 2")
        self._h = C.c_void_p()
        check(lib.hm_tree_build(locs.ctypes.data_as(C.c_void_p), locs.shape[0], int(leaf), float(eta),
                                C.byref(self._h)))
        cnt = np.zeros(6, dtype=np.int64)
        check(lib.hm_tree_counts(self._h, cnt.ctypes.data_as(C.c_void_p)))
        self.n, self.n_clusters, self.n_leaves, self.depth, self.n_blocks, self.n_admissible = map(int, cnt)

    def perm(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.int64)
        check(lib.hm_tree_perm(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def clusters(self) -> np.ndarray:
        out = np.empty((self.n_clusters, 4), dtype=np.int64)
        check(lib.hm_tree_clusters(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def blocks(self) -> np.ndarray:
        out = np.empty((self.n_blocks, 6), dtype=np.int64)
        check(lib.hm_tree_blocks(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def plan_summary(self, kmax: int = 160) -> dict:
        s = np.zeros(8)
        check(lib.hm_plan_dump(self._h, int(kmax), None, s.ctypes.data_as(C.c_void_p)))
        keys = ("pool_doubles", "slots", "chol_vm_tasks", "chol_trunc_tasks", "chol_waves", "chol_launches",
                "solve_waves", "solve_tasks")
        return dict(zip(keys, s.tolist()))

    def plan_dump(self, path: str, kmax: int = 160):
        check(lib.hm_plan_dump(self._h, int(kmax), path.encode(), None))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.hm_tree_free(h)
            self._h = None


# ---------------------------------------------------------------- dense check path
def dense_loglik(locs, theta, Z, device: int = 0, stream=None) -> np.ndarray:
    """Exact Eq. (1) on the GPU (n <= HM_DENSE_NMAX = 131072, 8 n^2 bytes of device
    memory).  Returns k x 3 (loglik, logdet, quad)."""
    if isinstance(locs, np.ndarray) or not hasattr(locs, "is_cuda"):
        locs = _as_f64(locs)
    if isinstance(Z, np.ndarray) or not hasattr(Z, "is_cuda"):
        Z = _as_f64(Z)
        if Z.ndim == 1:
            Z = Z[:, None]
        Z = np.asfortranarray(Z)
        n, k = Z.shape
        zp, zd = Z.ctypes.data_as(C.c_void_p), 0
    else:
        # torch tensors: 1-D (n,) or 2-D (k, n) contiguous == column-major n x k
        k, n = (Z.shape[0], Z.shape[1]) if Z.ndim == 2 else (1, Z.shape[0])
        zp, zd = ptr_of(Z)
    if n != int(locs.shape[0]):
        raise ValueError(f"Z has {n} rows, locations {int(locs.shape[0])}")
    lp, ld = ptr_of(locs)
    out = np.empty((k, 3), dtype=np.float64)
    check(lib.hm_dense_loglik(lp, ld, int(locs.shape[0]), Theta(*theta), zp, zd, int(k), int(device),
                              C.c_void_p(stream) if stream else None, out.ctypes.data_as(C.c_void_p)))
    return out


def matern_block(a, b, theta, device: int = 0) -> np.ndarray:
    a, b = _as_f64(a), _as_f64(b)
    out = np.empty((a.shape[0], b.shape[0]), dtype=np.float64, order="F")
    check(lib.hm_matern_block(a.ctypes.data_as(C.c_void_p), a.shape[0], b.ctypes.data_as(C.c_void_p),
                              b.shape[0], Theta(*theta), int(device), out.ctypes.data_as(C.c_void_p)))
    return out


# ---------------------------------------------------------------- H-matrix likelihood
def loglik_multi(handles, thetas, Zs):
    """hm_loglik_multi: handle i at thetas[i] on its own data Zs[i], all co-scheduled on
    one GPU.  Returns (len(handles) x k x 3 array, status code)."""
    nh = len(handles)
    keep = [_zarg(Z) for Z in Zs]
    ks = {kp[3] for kp in keep}
    devs = {kp[1] for kp in keep}
    if len(ks) != 1 or len(devs) != 1:
        raise ValueError("all data must have the same column count and location (host / device)")
    for H, kp, Z in zip(handles, keep, Zs):
        H._check_rows(kp[2], Z)
    k = ks.pop()
    hs = (C.c_void_p * nh)(*[H._h.value for H in handles])
    zp = (C.c_void_p * nh)(*[kp[0].value for kp in keep])
    th = np.ascontiguousarray(np.asarray(thetas, dtype=np.float64).reshape(nh, 3))
    out = np.empty((nh, k, 3))
    rc = lib.hm_loglik_multi(nh, hs, th.ctypes.data_as(C.c_void_p), zp, devs.pop(), int(k),
                             out.ctypes.data_as(C.c_void_p))
    return out, rc



def _zarg(Z):
    """(pointer, on_device, n, k, keepalive) for data vectors: numpy n / n x k, or torch (n,) / (k, n)."""
    if isinstance(Z, np.ndarray) or not hasattr(Z, "is_cuda"):
        Z = _as_f64(Z)
        if Z.ndim == 1:
            Z = Z[:, None]
        Z = np.asfortranarray(Z)
        return Z.ctypes.data_as(C.c_void_p), 0, Z.shape[0], Z.shape[1], Z
    k, n = (Z.shape[0], Z.shape[1]) if Z.ndim == 2 else (1, Z.shape[0])
    p, d = ptr_of(Z)
    return p, d, n, k, Z


class HMatrix:
    """C~(theta) in H-matrix format on one GPU (hm_build) and its H-Cholesky factor.

    PAPER.md Eq. (4): loglik(Z) = -n/2 log 2pi - sum log L~_ii - 1/2 v^T v with L~ v = Z.
    """

    def __init__(self, locs, theta, eps: float = 1e-8, leaf: int = 32, eta: float = 2.0, kmax: int = 160,
                 device: int = 0, stream=None, rel_eps: bool = False, coop_max: int = 0, eps_chol: float = 0.0,
                 exec_ctas: int = 0, adaptive_cap: bool = False):
        if isinstance(locs, np.ndarray) or not hasattr(locs, "is_cuda"):
            locs = _as_f64(locs)
        lp, ld = ptr_of(locs)
        self.n = int(locs.shape[0])
        self.device = int(device)
        self._h = C.c_void_p()
        self.params = Params(float(eps), int(leaf), float(eta), int(kmax), 1 if rel_eps else 0, int(coop_max),
                             float(eps_chol), int(exec_ctas), 1 if adaptive_cap else 0)
        rc = lib.hm_build(lp, ld, self.n, Theta(*theta), self.params, int(device),
                          C.c_void_p(stream) if stream else None, C.byref(self._h))
        check(rc)

    def assemble(self, theta):
        check(lib.hm_assemble(self._h, Theta(*theta)))

    def cholesky(self):
        check(lib.hm_cholesky(self._h))

    def _check_rows(self, n, Z):
        if n != self.n:
            raise ValueError(f"data has {n} rows, the H-matrix {self.n} (torch data is (n,) or (k, n))")
        if hasattr(Z, "is_cuda") and Z.is_cuda and Z.device.index != self.device:
            raise ValueError(f"data on {Z.device}, handle on cuda:{self.device}")

    def loglik(self, Z) -> np.ndarray:
        p, d, n, k, keep = _zarg(Z)
        self._check_rows(n, Z)
        out = np.empty((k, 3))
        check(lib.hm_loglik(self._h, p, d, int(k), out.ctypes.data_as(C.c_void_p)))
        return out

    def loglik_batch(self, thetas, Z):
        th = np.ascontiguousarray(np.asarray(thetas, dtype=np.float64).reshape(-1, 3))
        p, d, n, k, keep = _zarg(Z)
        self._check_rows(n, Z)
        out = np.empty((th.shape[0], k, 3))
        rc = lib.hm_loglik_batch(self._h, th.ctypes.data_as(C.c_void_p), th.shape[0], p, d, int(k),
                                 out.ctypes.data_as(C.c_void_p))
        return out, rc

    def set_batch_streams(self, streams: int):
        """Co-scheduled executors of loglik_batch (0 = default 4, 1 = sequential)."""
        check(lib.hm_set_batch_streams(self._h, int(streams)))

    def sample(self, xi) -> np.ndarray:
        p, d, n, k, keep = _zarg(xi)
        self._check_rows(n, xi)
        if d:
            raise TypeError("use a host array for xi (device variant: hm_sample with device pointers)")
        out = np.empty((n, k), order="F")
        check(lib.hm_sample(self._h, p, 0, int(k), out.ctypes.data_as(C.c_void_p), 0))
        return out

    def stats(self) -> dict:
        s = np.zeros(12)
        check(lib.hm_stats(self._h, s.ctypes.data_as(C.c_void_p)))
        keys = ("n", "dense_blocks", "lowrank_blocks", "max_rank_C", "max_rank_L", "bytes_C", "bytes_L",
                "compression_C", "chol_tasks", "chol_waves", "chol_launches", "max_trunc_width")
        return dict(zip(keys, s.tolist()))

    def timings(self) -> dict:
        s = np.zeros(3)
        check(lib.hm_timings(self._h, s.ctypes.data_as(C.c_void_p)))
        return dict(zip(("assemble_ms", "cholesky_ms", "loglik_ms"), s.tolist()))

    def profile(self, enable: bool):
        check(lib.hm_profile(self._h, 1 if enable else 0))

    KERNEL_FAMILIES = ("k_dense_gen", "k_aca", "k_trunc", "k_vm", "k_aux", "k_exec")

    def set_exec_grid(self, ctas: int):
        """Cap this handle's persistent executor at `ctas` CTAs (0 = all SMs), so
        several handles can run side by side on different streams."""
        check(lib.hm_set_exec_grid(self._h, int(ctas)))

    def set_exec_mode(self, mode: int):
        """2 = persistent ready-queue executor (default), 1 = persistent topological-claim
        executor, 0 = one launch per wave."""
        check(lib.hm_set_exec_mode(self._h, int(mode)))

    def trace(self, enable: bool, path: str | None = None):
        """Per-task executor timestamps (diagnostics); see hm_trace in include/hmlik.h."""
        check(lib.hm_trace(self._h, 1 if enable else 0, path.encode() if path else None))

    def checksum(self) -> np.ndarray:
        s = np.zeros(4)
        check(lib.hm_checksum(self._h, s.ctypes.data_as(C.c_void_p)))
        return s

    def to_dense(self) -> np.ndarray:
        """C~ (after assembly) or L~ (after cholesky) as a dense n x n array in the
        original point order (diagnostics; hm_to_dense)."""
        out = np.empty((self.n, self.n), order="F")
        check(lib.hm_to_dense(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def kernel_stats(self) -> dict:
        s = np.zeros(24)
        check(lib.hm_kernel_stats(self._h, s.ctypes.data_as(C.c_void_p)))
        return {k: dict(launches=s[4 * i], ms=s[4 * i + 1], flops=s[4 * i + 2], bytes=s[4 * i + 3])
                for i, k in enumerate(self.KERNEL_FAMILIES)}

    def close(self):
        if getattr(self, "_h", None):
            lib.hm_free(self._h)
            self._h = None

    def __del__(self):
        self.close()
