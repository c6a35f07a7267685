"""B200-native MRA log-likelihood (arXiv:1905.00141) -- thin Python binding of libmra_b200.so.

Argument marshalling only: every evaluation step runs in the library's sm_100a kernels
(include/mra.h). The functions carry the C-ABI names:

    mra_plan_create(x, y, M, J, r, **opts) -> handle
    mra_loglik(plan, y_host, theta, posterior=False, regions=False)
    mra_loglik_dev(plan, y_tensor_cuda, theta, ...)
    mra_loglik_batch_dev(plan, y_tensor_cuda, thetas)
    mra_shard_size / mra_loglik_shard / mra_loglik_finish       (multi-GPU subtree sharding)
    mra_plan_info / mra_plan_layout / mra_last_launches / mra_plan_destroy

theta = (cov, sigma2, rho, tau2) with cov 0 = exponential, 1 = Matern-3/2.
There is no CPU fallback: if the CUDA library is missing or no GPU is visible these raise.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmra_b200.so")

COV_EXP = 0
COV_MATERN32 = 1
E_OVER_100 = math.e / 100.0


class MraError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"mra status {status}: {msg}")
        self.status = status


class _Theta(ctypes.Structure):
    _fields_ = [("cov", ctypes.c_int), ("sigma2", ctypes.c_double), ("rho", ctypes.c_double),
                ("tau2", ctypes.c_double)]


_DALLOC = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p)
_DFREE = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p)


class _Opts(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_double), ("xscale", ctypes.c_double), ("yscale", ctypes.c_double),
                ("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("rank", ctypes.c_int),
                ("world", ctypes.c_int), ("shard_level", ctypes.c_int), ("mem_budget_gb", ctypes.c_double),
                ("wide", ctypes.c_int), ("host_plan", ctypes.c_int), ("stream_prior", ctypes.c_int),
                ("theta_lanes", ctypes.c_int), ("nccl_id", ctypes.c_void_p), ("dalloc", _DALLOC),
                ("dfree", _DFREE), ("graph", ctypes.c_int)]


class _Post(ctypes.Structure):
    _fields_ = [("mu", ctypes.c_void_p), ("smooth", ctypes.c_void_p), ("region_d", ctypes.c_void_p),
                ("region_u", ctypes.c_void_p), ("d", ctypes.c_double), ("u", ctypes.c_double)]


_lib = None
EXPORTS = ["mra_plan_create", "mra_loglik", "mra_loglik_dev", "mra_loglik_batch_dev", "mra_loglik_batch", "mra_predict", "mra_optimize", "mra_shard_size",
           "mra_loglik_shard", "mra_loglik_finish", "mra_mutop_size", "mra_loglik_shard_post",
           "mra_loglik_finish_post", "mra_posterior_shard", "mra_plan_info", "mra_plan_layout", "mra_plan_shards", "mra_plan_memory",
           "mra_profile", "mra_kernel_times", "mra_last_launches", "mra_plan_destroy", "mra_last_error",
           "mra_nccl_unique_id"]


def load_library(path: str = LIB_PATH):
    """dlopen libmra_b200.so and declare the C-ABI signatures (no GPU needed to load)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -m paper_1905_00141_b200.build` "
                           "(nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    D = ctypes.POINTER(ctypes.c_double)
    U64 = ctypes.c_uint64
    lib.mra_plan_create.restype = ctypes.c_int
    lib.mra_plan_create.argtypes = [D, D, U64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(_Opts), ctypes.POINTER(P)]
    lib.mra_loglik.restype = ctypes.c_int
    lib.mra_loglik.argtypes = [P, D, ctypes.POINTER(_Theta), D, ctypes.POINTER(_Post)]
    lib.mra_loglik_dev.restype = ctypes.c_int
    lib.mra_loglik_dev.argtypes = [P, P, ctypes.POINTER(_Theta), D, ctypes.POINTER(_Post)]
    lib.mra_loglik_batch_dev.restype = ctypes.c_int
    lib.mra_loglik_batch_dev.argtypes = [P, P, ctypes.POINTER(_Theta), ctypes.c_int, D]
    lib.mra_loglik_batch.restype = ctypes.c_int
    lib.mra_loglik_batch.argtypes = [P, D, ctypes.POINTER(_Theta), ctypes.c_int, D]
    lib.mra_shard_size.restype = U64
    lib.mra_shard_size.argtypes = [P]
    lib.mra_loglik_shard.restype = ctypes.c_int
    lib.mra_loglik_shard.argtypes = [P, P, ctypes.POINTER(_Theta), P]
    lib.mra_mutop_size.restype = U64
    lib.mra_mutop_size.argtypes = [P]
    lib.mra_loglik_shard_post.restype = ctypes.c_int
    lib.mra_loglik_shard_post.argtypes = [P, P, ctypes.POINTER(_Theta), P]
    lib.mra_loglik_finish_post.restype = ctypes.c_int
    lib.mra_loglik_finish_post.argtypes = [P, ctypes.POINTER(_Theta), P, D, P]
    lib.mra_posterior_shard.restype = ctypes.c_int
    lib.mra_posterior_shard.argtypes = [P, P, P, P]
    lib.mra_loglik_finish.restype = ctypes.c_int
    lib.mra_loglik_finish.argtypes = [P, ctypes.POINTER(_Theta), P, D]
    lib.mra_plan_info.restype = ctypes.c_int
    lib.mra_plan_info.argtypes = [P, ctypes.POINTER(U64), ctypes.POINTER(ctypes.c_int), ctypes.POINTER(U64),
                                  ctypes.POINTER(U64), ctypes.POINTER(U64), ctypes.POINTER(U64)]
    lib.mra_plan_layout.restype = ctypes.c_int
    lib.mra_plan_layout.argtypes = [P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64), D, D]
    lib.mra_plan_shards.restype = ctypes.c_int
    lib.mra_plan_shards.argtypes = [P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(U64)]
    lib.mra_plan_memory.restype = ctypes.c_int
    lib.mra_plan_memory.argtypes = [P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), ctypes.POINTER(U64),
                                    ctypes.POINTER(U64)]
    lib.mra_profile.restype = ctypes.c_int
    lib.mra_profile.argtypes = [P, ctypes.c_int]
    lib.mra_optimize.restype = ctypes.c_int
    lib.mra_optimize.argtypes = [P, P, ctypes.POINTER(_Theta), D, D, ctypes.c_int, ctypes.c_double, D,
                                 ctypes.POINTER(ctypes.c_int)]
    lib.mra_predict.restype = ctypes.c_int
    lib.mra_predict.argtypes = [P, D, D, U64, D, D]
    lib.mra_kernel_times.restype = ctypes.c_int
    lib.mra_kernel_times.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(U64)]
    lib.mra_last_launches.restype = U64
    lib.mra_last_launches.argtypes = [P]
    lib.mra_plan_destroy.restype = None
    lib.mra_plan_destroy.argtypes = [P]
    lib.mra_last_error.restype = ctypes.c_char_p
    lib.mra_last_error.argtypes = []
    lib.mra_nccl_unique_id.restype = ctypes.c_int
    lib.mra_nccl_unique_id.argtypes = [P]
    _lib = lib
    return lib


def _check(status):
    if status != 0:
        raise MraError(status, _lib.mra_last_error().decode())


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _theta(theta):
    cov, s2, rho, t2 = theta
    return _Theta(int(cov), float(s2), float(rho), float(t2))


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


class PlanHandle:
    """Owning handle of an mra_plan (destroyed on close / garbage collection)."""

    def __init__(self, ptr, n, M, J, r, keep=()):
        self.ptr = ptr
        self._keep = keep            # allocator-hook callbacks must outlive the plan
        self.n, self.M, self.J, self.r = n, M, J, r
        info = mra_plan_info(self)
        self.n_retained = info["n_retained"]
        self.r_hat = info["r_hat"]
        self.n_regions = info["n_regions"]
        self.n_leaves = info["n_leaves"]
        self.n_interior = self.n_regions - self.n_leaves

    def close(self):
        if self.ptr:
            _lib.mra_plan_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mra_nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (create on rank 0, send to every rank, pass as nccl_id=)."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(lib.mra_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


def _torch_hooks():
    """Allocator hooks that take the plan's device memory from torch's caching allocator."""
    import torch

    def _alloc(nbytes, device, stream):
        try:
            with torch.cuda.device(device):
                return torch.cuda.caching_allocator_alloc(int(nbytes), device, stream or 0)
        except Exception:
            return None

    def _free(ptr, device, stream):
        torch.cuda.caching_allocator_delete(ptr)

    return _DALLOC(_alloc), _DFREE(_free)


def mra_plan_create(x, y, M, J, r, offset=0.0, xscale=0.0, yscale=0.0, device=-1, stream=None, rank=0,
                    world=1, shard_level=0, mem_budget_gb=0.0, wide=0, host_plan=0,
                    stream_prior=0, theta_lanes=0, nccl_id=None, torch_alloc=False, graph=False) -> PlanHandle:
    """Build a plan. nccl_id (bytes from mra_nccl_unique_id on rank 0) gives the plan its own NCCL communicator
    for the in-library exchange step of subtree sharding; torch_alloc=True routes its device memory through
    torch's caching allocator (opts.dalloc / dfree)."""
    lib = load_library()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if x.shape != y.shape or x.ndim != 1:
        raise ValueError("x and y must be 1-D arrays of equal length")
    idbuf = None
    if nccl_id is not None:
        if len(nccl_id) != 128:
            raise ValueError("nccl_id must be the 128 bytes of an ncclUniqueId")
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
    hooks = _torch_hooks() if torch_alloc else (_DALLOC(), _DFREE())
    opts = _Opts(float(offset), float(xscale), float(yscale), int(device), _stream_ptr(stream), int(rank),
                 int(world), int(shard_level), float(mem_budget_gb), int(wide), int(host_plan), int(stream_prior),
                 int(theta_lanes), ctypes.cast(idbuf, ctypes.c_void_p) if idbuf is not None else None,
                 hooks[0], hooks[1], int(bool(graph)))
    out = ctypes.c_void_p()
    _check(lib.mra_plan_create(_dptr(x), _dptr(y), x.shape[0], int(M), int(J), int(r), ctypes.byref(opts),
                               ctypes.byref(out)))
    return PlanHandle(out.value, x.shape[0], M, J, r, keep=hooks if torch_alloc else ())


def _post_struct(plan, posterior, regions, host, device=None):
    bufs = {}
    post = _Post()
    if posterior:
        nmu = max(1, plan.n_interior * plan.r_hat)
        if host:
            bufs["mu"] = np.empty(nmu)
            bufs["smooth"] = np.empty(plan.n)
            post.mu = bufs["mu"].ctypes.data
            post.smooth = bufs["smooth"].ctypes.data
        else:
            import torch
            bufs["mu"] = torch.empty(nmu, dtype=torch.float64, device=device)
            bufs["smooth"] = torch.empty(plan.n, dtype=torch.float64, device=device)
            post.mu = bufs["mu"].data_ptr()
            post.smooth = bufs["smooth"].data_ptr()
    if regions:
        bufs["region_d"] = np.empty(plan.n_regions)
        bufs["region_u"] = np.empty(plan.n_regions)
        post.region_d = bufs["region_d"].ctypes.data
        post.region_u = bufs["region_u"].ctypes.data
    return post, bufs


def _result(plan, ll, post, bufs, posterior):
    out = {"loglik": ll.value, "d": post.d, "u": post.u, "n_retained": plan.n_retained}
    if "region_d" in bufs:
        out["region_d"], out["region_u"] = bufs["region_d"], bufs["region_u"]
    if posterior:
        out["mu"] = bufs["mu"][: plan.n_interior * plan.r_hat].reshape(plan.n_interior, plan.r_hat)
        out["smooth"] = bufs["smooth"]
    return out


def mra_loglik(plan: PlanHandle, y, theta, posterior=False, regions=False):
    """Host y (original order) -> dict(loglik, d, u[, region_d, region_u][, mu, smooth])."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    if y.shape[0] != plan.n:
        raise ValueError("y has the wrong length")
    th = _theta(theta)
    ll = ctypes.c_double()
    post, bufs = _post_struct(plan, posterior, regions, host=True)
    _check(_lib.mra_loglik(plan.ptr, _dptr(y), ctypes.byref(th), ctypes.byref(ll), ctypes.byref(post)))
    return _result(plan, ll, post, bufs, posterior)


def _check_dev(t, n, what="y_dev"):
    """A device buffer handed to the library: contiguous float64 CUDA memory of at least n values."""
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{what} must be a contiguous torch.float64 CUDA tensor")
    if t.numel() < n:
        raise ValueError(f"{what} holds {t.numel()} values, the call needs {n}")


def mra_loglik_dev(plan: PlanHandle, y_dev, theta, posterior=False, regions=False):
    """y_dev: torch float64 CUDA tensor (original order). Posterior outputs stay on the device."""
    _check_dev(y_dev, plan.n)
    th = _theta(theta)
    ll = ctypes.c_double()
    post, bufs = _post_struct(plan, posterior, regions, host=False, device=y_dev.device)
    _check(_lib.mra_loglik_dev(plan.ptr, ctypes.c_void_p(y_dev.data_ptr()), ctypes.byref(th), ctypes.byref(ll),
                               ctypes.byref(post)))
    return _result(plan, ll, post, bufs, posterior)


def mra_loglik_batch_dev(plan: PlanHandle, y_dev, thetas):
    _check_dev(y_dev, plan.n)
    arr = (_Theta * len(thetas))(*[_theta(t) for t in thetas])
    out = np.empty(len(thetas))
    _check(_lib.mra_loglik_batch_dev(plan.ptr, ctypes.c_void_p(y_dev.data_ptr()), arr, len(thetas), _dptr(out)))
    return out


def mra_loglik_batch(plan: PlanHandle, y, thetas):
    """Likelihood sweep with y a host array (copied to the device once)."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    if y.shape != (plan.n,):
        raise ValueError("y must have one value per input location")
    arr = (_Theta * len(thetas))(*[_theta(t) for t in thetas])
    out = np.empty(len(thetas))
    _check(_lib.mra_loglik_batch(plan.ptr, _dptr(y), arr, len(thetas), _dptr(out)))
    return out


def mra_shard_size(plan: PlanHandle) -> int:
    return int(_lib.mra_shard_size(plan.ptr))


def mra_loglik_shard(plan: PlanHandle, y_dev, theta, xbuf_dev):
    _check_dev(y_dev, plan.n)
    _check_dev(xbuf_dev, mra_shard_size(plan), "xbuf_dev")
    th = _theta(theta)
    _check(_lib.mra_loglik_shard(plan.ptr, ctypes.c_void_p(y_dev.data_ptr()), ctypes.byref(th),
                                 ctypes.c_void_p(xbuf_dev.data_ptr())))


def mra_mutop_size(plan: PlanHandle) -> int:
    return int(_lib.mra_mutop_size(plan.ptr))


def mra_loglik_shard_post(plan: PlanHandle, y_dev, theta, xbuf_dev):
    _check_dev(y_dev, plan.n)
    _check_dev(xbuf_dev, mra_shard_size(plan), "xbuf_dev")
    th = _theta(theta)
    _check(_lib.mra_loglik_shard_post(plan.ptr, ctypes.c_void_p(y_dev.data_ptr()), ctypes.byref(th),
                                      ctypes.c_void_p(xbuf_dev.data_ptr())))


def mra_loglik_finish_post(plan: PlanHandle, theta, xbuf_dev, mutop_dev) -> float:
    _check_dev(xbuf_dev, mra_shard_size(plan), "xbuf_dev")
    _check_dev(mutop_dev, mra_mutop_size(plan), "mutop_dev")
    th = _theta(theta)
    ll = ctypes.c_double()
    _check(_lib.mra_loglik_finish_post(plan.ptr, ctypes.byref(th), ctypes.c_void_p(xbuf_dev.data_ptr()),
                                       ctypes.byref(ll), ctypes.c_void_p(mutop_dev.data_ptr())))
    return ll.value


def mra_posterior_shard(plan: PlanHandle, mutop_dev, mu_dev=None, smooth_dev=None):
    _check_dev(mutop_dev, mra_mutop_size(plan), "mutop_dev")
    if mu_dev is not None:
        _check_dev(mu_dev, plan.n_interior * plan.r_hat, "mu_dev")
    if smooth_dev is not None:
        _check_dev(smooth_dev, plan.n, "smooth_dev")
    _check(_lib.mra_posterior_shard(plan.ptr, ctypes.c_void_p(mutop_dev.data_ptr()),
                                    ctypes.c_void_p(mu_dev.data_ptr() if mu_dev is not None else 0),
                                    ctypes.c_void_p(smooth_dev.data_ptr() if smooth_dev is not None else 0)))


def mra_loglik_finish(plan: PlanHandle, theta, xbuf_dev) -> float:
    _check_dev(xbuf_dev, mra_shard_size(plan), "xbuf_dev")
    th = _theta(theta)
    ll = ctypes.c_double()
    _check(_lib.mra_loglik_finish(plan.ptr, ctypes.byref(th), ctypes.c_void_p(xbuf_dev.data_ptr()),
                                  ctypes.byref(ll)))
    return ll.value


def mra_plan_info(plan: PlanHandle) -> dict:
    v = [ctypes.c_uint64() for _ in range(5)]
    rh = ctypes.c_int()
    _check(_lib.mra_plan_info(plan.ptr, ctypes.byref(v[0]), ctypes.byref(rh), ctypes.byref(v[1]),
                              ctypes.byref(v[2]), ctypes.byref(v[3]), ctypes.byref(v[4])))
    return dict(n_retained=v[0].value, r_hat=rh.value, n_regions=v[1].value, n_leaves=v[2].value,
                n_empty_leaves=v[3].value, max_leaf=v[4].value)


def mra_plan_layout(plan: PlanHandle) -> dict:
    perm = np.empty(plan.n_retained, dtype=np.int64)
    off = np.empty(plan.n_leaves + 1, dtype=np.int64)
    nk = max(1, plan.n_interior * plan.r_hat)
    kx = np.empty(nk)
    ky = np.empty(nk)
    _check(_lib.mra_plan_layout(plan.ptr, perm.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _dptr(kx), _dptr(ky)))
    return dict(perm=perm, leaf_off=off, knots_x=kx[: plan.n_interior * plan.r_hat],
                knots_y=ky[: plan.n_interior * plan.r_hat])


def mra_plan_shards(plan: PlanHandle) -> dict:
    lvl = ctypes.c_int()
    n = ctypes.c_uint64()
    _check(_lib.mra_plan_shards(plan.ptr, ctypes.byref(lvl), None, ctypes.byref(n)))
    own = np.empty(max(1, n.value), dtype=np.int64)
    _check(_lib.mra_plan_shards(plan.ptr, ctypes.byref(lvl), own.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                ctypes.byref(n)))
    return dict(shard_level=lvl.value, own=own[: n.value])


def mra_plan_memory(plan: PlanHandle) -> dict:
    """Device-memory layout: streamed prior (NEXT-4), chunk level / size, bytes held."""
    sp, cl = ctypes.c_int(), ctypes.c_int()
    kc, nb = ctypes.c_uint64(), ctypes.c_uint64()
    _check(_lib.mra_plan_memory(plan.ptr, ctypes.byref(sp), ctypes.byref(cl), ctypes.byref(kc), ctypes.byref(nb)))
    return dict(streams_prior=bool(sp.value), chunk_level=cl.value, chunk_regions=kc.value, device_bytes=nb.value)


def mra_profile(plan: PlanHandle, enable: bool = True):
    _check(_lib.mra_profile(plan.ptr, int(bool(enable))))


KERNEL_CLASSES = ("prior", "bottom", "merge", "other", "chain", "sigma", "factor", "solve", "syrk_merge", "covgen")


def mra_kernel_times(plan: PlanHandle) -> dict:
    """Accumulated device ms and launch counts per kernel class since mra_profile(plan, True)."""
    ms = (ctypes.c_double * len(KERNEL_CLASSES))()
    cnt = (ctypes.c_uint64 * len(KERNEL_CLASSES))()
    _check(_lib.mra_kernel_times(plan.ptr, ms, cnt))
    return {k: (ms[i], cnt[i]) for i, k in enumerate(KERNEL_CLASSES)}


def mra_optimize(plan: PlanHandle, y_dev, theta0, lower=None, upper=None, max_evals=200, tol=1e-6):
    """Maximise log L over (sigma2, rho, tau2) from theta0 = (cov, sigma2, rho, tau2); y_dev a CUDA tensor.
    Returns (theta, loglik, n_evals)."""
    _check_dev(y_dev, plan.n)
    th = _Theta(int(theta0[0]), float(theta0[1]), float(theta0[2]), float(theta0[3]))
    D = ctypes.POINTER(ctypes.c_double)
    lo = None if lower is None else (ctypes.c_double * 3)(*[float(v) for v in lower])
    hi = None if upper is None else (ctypes.c_double * 3)(*[float(v) for v in upper])
    ll = ctypes.c_double()
    ne = ctypes.c_int()
    _check(_lib.mra_optimize(plan.ptr, ctypes.c_void_p(y_dev.data_ptr()), ctypes.byref(th),
                             ctypes.cast(lo, D) if lo is not None else None,
                             ctypes.cast(hi, D) if hi is not None else None, int(max_evals), float(tol),
                             ctypes.byref(ll), ctypes.byref(ne)))
    return (th.cov, th.sigma2, th.rho, th.tau2), ll.value, ne.value


def mra_predict(plan: PlanHandle, qx, qy):
    """Posterior mean / variance of X at query points (host arrays) for the last evaluation, which
    must have requested posterior state (posterior=True). NaN outside the root domain."""
    qx = np.ascontiguousarray(qx, dtype=np.float64)
    qy = np.ascontiguousarray(qy, dtype=np.float64)
    if qx.shape != qy.shape or qx.ndim != 1:
        raise ValueError("qx, qy must be 1-D arrays of equal length")
    mean = np.empty(qx.shape[0])
    var = np.empty(qx.shape[0])
    D = ctypes.POINTER(ctypes.c_double)
    _check(_lib.mra_predict(plan.ptr, qx.ctypes.data_as(D), qy.ctypes.data_as(D), qx.shape[0],
                            mean.ctypes.data_as(D), var.ctypes.data_as(D)))
    return mean, var


def mra_last_launches(plan: PlanHandle) -> int:
    return int(_lib.mra_last_launches(plan.ptr))


def mra_plan_destroy(plan: PlanHandle):
    plan.close()


def atilde_bound_gib(J, M, r):
    """Eq. (1) of PAPER.md:486-488: upper bound of the paper's ATilde memory, J^{M-1} M (M-1) r^2 2^-28 GiB."""
    return J ** (M - 1) * M * (M - 1) * r * r * 2.0 ** -28
