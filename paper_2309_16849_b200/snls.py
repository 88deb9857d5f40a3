"""Python front end over the C-ABI (include/snls_cuda.h) -- the same operator surface as the
reference's C++ API (search.hpp:126-158, aggregate.hpp:22-85), on torch CUDA tensors.

torch is only the device-memory / stream plumbing here: every operation is one or more of
the hand-written sm_100a kernels in libsnls_cuda.so, called through ctypes.  There is no
CPU fallback: if the library or a B200 is missing the calls raise.

Error behaviour mirrors the reference: configuration problems raise ConfigError and domain
problems DomainError (errors.hpp:9-17) with the reference's messages.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field
from typing import Optional

PKG = os.path.dirname(os.path.abspath(__file__))
# SNLS_LIB_OVERRIDE: an A/B build of the same library (scripts/build_variant.sh)
LIB_PATH = os.environ.get("SNLS_LIB_OVERRIDE") or os.path.join(PKG, "libsnls_cuda.so")

METRIC_IP, METRIC_L2 = 0, 1
MODE_FUSED, MODE_FULLGRID = 0, 1


class SnlsError(RuntimeError):
    pass


class ConfigError(SnlsError):
    """snls::ConfigError (errors.hpp:9-12)."""


class DomainError(SnlsError):
    """snls::DomainError (errors.hpp:14-17)."""


class CudaError(SnlsError):
    pass


class IoError(SnlsError):
    """snls::IoError (errors.hpp): file formats."""


@dataclass
class SearchConfig:
    """snls::SearchConfig (search.hpp:17-35)."""

    ws: int = 9
    wt: int = 0
    ps: int = 1
    stride0: int = 1
    stride1: float = 1.0
    topl: int = 1
    metric: str = "l2"  # 'ip' (inner product) or 'l2' (negated squared L2)
    softmax_scale: float = 1.0

    def window_frames(self) -> int:
        return 2 * self.wt + 1

    def window_slots(self) -> int:
        return self.window_frames() * self.ws * self.ws

    def hole_free(self) -> bool:
        return (self.ps - 1) // 2 < self.stride0

    def chain_stride(self) -> int:
        return max(self.wt - 1, 0)


class _Config(C.Structure):
    _fields_ = [("ws", C.c_int), ("wt", C.c_int), ("ps", C.c_int), ("stride0", C.c_int),
                ("stride1", C.c_double), ("topl", C.c_int), ("metric", C.c_int),
                ("softmax_scale", C.c_double)]


class _Dims(C.Structure):
    _fields_ = [("t", C.c_int), ("h", C.c_int), ("w", C.c_int), ("f", C.c_int)]


def _cfg(c: SearchConfig) -> _Config:
    if c.metric not in ("ip", "l2"):
        raise ConfigError("SearchConfig: unknown metric")
    return _Config(int(c.ws), int(c.wt), int(c.ps), int(c.stride0), float(c.stride1), int(c.topl),
                   METRIC_IP if c.metric == "ip" else METRIC_L2, float(c.softmax_scale))


_lib = None
_lib_lock = threading.Lock()
VOIDP = C.c_void_p


def lib() -> C.CDLL:
    """Load libsnls_cuda.so (raises if it has not been built: no silent fallback)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise CudaError(f"{LIB_PATH} is missing; build it with "
                                "`python -m paper_2309_16849_b200.build`")
            L = C.CDLL(LIB_PATH)
            L.snls_last_error.restype = C.c_char_p
            L.snls_uniform_fill_f32.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_int64, VOIDP]
            L.snls_query_grid.argtypes = [_Dims, C.c_int, C.POINTER(C.c_int64),
                                          C.POINTER(C.c_int), C.POINTER(C.c_int)]
            L.snls_ctx_create.argtypes = [C.c_int, VOIDP, C.POINTER(VOIDP)]
            L.snls_ctx_destroy.argtypes = [VOIDP]
            L.snls_ctx_set_stream.argtypes = [VOIDP, VOIDP]
            L.snls_ctx_sync_check.argtypes = [VOIDP]
            L.snls_ctx_launch_count.argtypes = [VOIDP, C.POINTER(C.c_int64)]
            L.snls_ctx_last_search_path.argtypes = [VOIDP, C.POINTER(C.c_int)]
            L.snls_ctx_force_generic.argtypes = [VOIDP, C.c_int]
            L.snls_ctx_set_search_kernel.argtypes = [VOIDP, C.c_int]
            if hasattr(L, "snls_ctx_set_search_band"):
                L.snls_ctx_set_search_band.argtypes = [VOIDP, C.c_int]
            L.snls_validate_config.argtypes = [C.POINTER(_Config)]
            P = C.POINTER(_Config)
            L.snls_search_fwd.argtypes = [VOIDP, P, _Dims, VOIDP, VOIDP, VOIDP, VOIDP, C.c_int,
                                          VOIDP, VOIDP, VOIDP, VOIDP]
            L.snls_search_fwd_frames.argtypes = [VOIDP, P, _Dims, C.c_int, C.c_int, VOIDP, VOIDP,
                                                 VOIDP, VOIDP, C.c_int, VOIDP, VOIDP, VOIDP, VOIDP]
            L.snls_wpsum_fwd_frames.argtypes = [VOIDP, P, _Dims, C.c_int, C.c_int, VOIDP, VOIDP,
                                                VOIDP, VOIDP, VOIDP]
            L.snls_search_grid.argtypes = [VOIDP, P, _Dims, VOIDP, VOIDP, VOIDP, VOIDP, VOIDP, VOIDP]
            L.snls_topl.argtypes = [VOIDP, C.c_int64, C.c_int, VOIDP, VOIDP, C.c_int, VOIDP, VOIDP]
            L.snls_replay.argtypes = [VOIDP, P, _Dims, VOIDP, VOIDP, VOIDP, VOIDP]
            L.snls_search_bwd.argtypes = [VOIDP, P, _Dims, VOIDP, VOIDP, VOIDP, VOIDP, VOIDP,
                                          VOIDP, VOIDP, VOIDP, VOIDP]
            L.snls_softmax_rows.argtypes = [VOIDP, C.c_int64, C.c_int, C.c_double, VOIDP, VOIDP]
            L.snls_wpsum_fwd.argtypes = [VOIDP, P, _Dims, VOIDP, VOIDP, VOIDP, VOIDP, VOIDP]
            L.snls_gather_stack.argtypes = [VOIDP, P, _Dims, VOIDP, VOIDP, VOIDP, VOIDP]
            L.snls_wpsum_bwd.argtypes = [VOIDP, P, _Dims, VOIDP, VOIDP, VOIDP, VOIDP, VOIDP,
                                         VOIDP, VOIDP]
            L.snls_ctx_get_stream.argtypes = [VOIDP, C.POINTER(VOIDP)]
            L.snls_raw_info.argtypes = [C.c_char_p, C.POINTER(_Dims), C.POINTER(C.c_int)]
            L.snls_raw_read.argtypes = [C.c_char_p, VOIDP, C.c_int64]
            L.snls_raw_write.argtypes = [C.c_char_p, _Dims, VOIDP, C.c_int]
            L.snls_flo_read.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), VOIDP]
            L.snls_flo_write.argtypes = [C.c_char_p, C.c_int, C.c_int, VOIDP]
            L.snls_block_match.argtypes = [VOIDP, _Dims, VOIDP, VOIDP, C.c_int, C.c_int, VOIDP]
            L.snls_psnr_frames.argtypes = [VOIDP, _Dims, VOIDP, VOIDP, C.c_double, VOIDP]
            L.snls_gaussian_noise_f32.argtypes = [C.c_uint64, C.c_double, C.c_int64, VOIDP, VOIDP]
            L.snls_align_frames.argtypes = [VOIDP, P, _Dims, VOIDP, C.c_double, C.c_uint64, C.c_int,
                                            VOIDP, C.c_int, C.c_int, VOIDP, VOIDP, VOIDP, VOIDP]
            L.snls_search_bwd_frames.argtypes = [VOIDP, P, _Dims, C.c_int, C.c_int] + [VOIDP] * 9
            if hasattr(L, "snls_train_bwd"):
                L.snls_train_bwd.argtypes = [VOIDP, P, _Dims] + [VOIDP] * 17 + [C.c_int]
            if hasattr(L, "snls_replay64"):
                L.snls_replay64.argtypes = [VOIDP, P, _Dims, C.c_int, C.c_int, VOIDP, VOIDP, VOIDP, C.c_int, VOIDP]
            if hasattr(L, "snls_search_bwd_ex"):  # (absent from A/B builds of older trees)
                L.snls_search_bwd_ex.argtypes = [VOIDP, P, _Dims, C.c_int, C.c_int] + [VOIDP] * 11 + [C.c_int]
                L.snls_search_tape64.argtypes = [VOIDP, P, _Dims, C.c_int, C.c_int] + [VOIDP] * 5
            L.snls_wpsum_bwd_frames.argtypes = [VOIDP, P, _Dims, C.c_int, C.c_int] + [VOIDP] * 7
            if hasattr(L, "snls_wpsum_bwd_ex"):
                L.snls_wpsum_bwd_ex.argtypes = [VOIDP, P, _Dims, C.c_int, C.c_int] + [VOIDP] * 7 + [C.c_int]
            L.snls_host_register.argtypes = [VOIDP, C.c_uint64]
            L.snls_host_unregister.argtypes = [VOIDP]
            L.snls_pipeline_create.argtypes = [VOIDP, P, _Dims, C.c_int, C.POINTER(VOIDP)]
            L.snls_pipeline_destroy.argtypes = [VOIDP]
            L.snls_pipeline_run.argtypes = [VOIDP] + [VOIDP] * 10
            L.snls_pipeline_submit.argtypes = [VOIDP] + [VOIDP] * 10
            L.snls_pipeline_wait.argtypes = [VOIDP]
            _lib = L
        return _lib


def _raise(rc: int):
    if rc == 0:
        return
    msg = lib().snls_last_error().decode()
    if rc == 1:
        raise ConfigError(msg)
    if rc == 2:
        raise DomainError(msg)
    if rc == 3:
        raise CudaError(msg)
    if rc == 5:
        raise IoError(msg)
    raise SnlsError(msg)


def validate(cfg: SearchConfig) -> None:
    """SearchConfig::validate (search.cpp:21-32) -- host only, no device needed."""
    c = _cfg(cfg)
    _raise(lib().snls_validate_config(C.byref(c)))


def query_grid(t: int, h: int, w: int, stride0: int):
    rows, nh, nw = C.c_int64(), C.c_int(), C.c_int()
    _raise(lib().snls_query_grid(_Dims(t, h, w, 1), stride0, C.byref(rows), C.byref(nh), C.byref(nw)))
    return rows.value, nh.value, nw.value


def uniform_fill(seed: int, lo: float, hi: float, n: int):
    """UniformStream(seed).next_in(lo, hi) (rng.hpp:12-24) as float32 numpy, host side."""
    import numpy as np

    out = np.empty(n, np.float32)
    _raise(lib().snls_uniform_fill_f32(C.c_uint64(seed), lo, hi, n, out.ctypes.data))
    return out


# ---------------------------------------------------------------------------------------
class Context:
    """One snls_ctx per (device, stream)."""

    def __init__(self, device: int = 0, stream=None):
        import torch

        self.torch = torch
        self.device = device
        s = stream if stream is not None else torch.cuda.current_stream(device)
        self.stream = s
        h = VOIDP()
        _raise(lib().snls_ctx_create(device, VOIDP(s.cuda_stream), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib().snls_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream):
        self.stream = stream
        _raise(lib().snls_ctx_set_stream(self.h, VOIDP(stream.cuda_stream)))

    def sync_check(self):
        _raise(lib().snls_ctx_sync_check(self.h))

    def launch_count(self) -> int:
        n = C.c_int64()
        _raise(lib().snls_ctx_launch_count(self.h, C.byref(n)))
        return n.value

    def last_search_path(self) -> int:
        n = C.c_int()
        _raise(lib().snls_ctx_last_search_path(self.h, C.byref(n)))
        return n.value

    def force_generic(self, on: bool):
        _raise(lib().snls_ctx_force_generic(self.h, int(on)))

    def set_search_band(self, band: int):
        """-1 auto, 0 plain raster, > 0 query rows per band (snls_ctx_set_search_band)."""
        _raise(lib().snls_ctx_set_search_band(self.h, int(band)))

    def set_search_kernel(self, kind: str):
        """'auto' | 'tiled' | 'stream' register plan for the stride1 == 1 search."""
        _raise(lib().snls_ctx_set_search_kernel(self.h, {"auto": 0, "tiled": 1, "stream": 2}[kind]))


_ctxs: dict = {}


def context(device: Optional[int] = None) -> Context:
    import torch

    dev = torch.cuda.current_device() if device is None else device
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    if key not in _ctxs:
        _ctxs[key] = Context(dev, torch.cuda.current_stream(dev))
    return _ctxs[key]


def _ptr(t):
    if t is None:
        return None
    import torch

    if not t.is_cuda:
        raise SnlsError("snls: tensors must live on a CUDA device")
    if not t.is_contiguous():
        raise SnlsError("snls: tensors must be contiguous")
    if t.dtype not in (torch.float32, torch.int32, torch.float64):
        raise SnlsError(f"snls: unsupported dtype {t.dtype}")
    if t.data_ptr() % 16:
        # the kernels load float4 vectors from the base pointers: a misaligned view would
        # fault (and a misaligned-address fault poisons the whole CUDA context)
        raise SnlsError("snls: tensor storage must be 16-byte aligned (use .clone() on a view)")
    return VOIDP(t.data_ptr())


def _dims(v) -> _Dims:
    if v.dim() != 4:
        raise DomainError("snls: videos are T x H x W x F")
    t, h, w, f = v.shape
    return _Dims(t, h, w, f)


@dataclass
class SearchResult:
    """snls::SearchResult (search.hpp:112-116) with the device tape (see snls_cuda.h)."""

    sims: object
    offsets: object
    chains: object = None
    weights: object = None
    cfg: SearchConfig = field(default_factory=SearchConfig)

    def centers(self):
        """Absolute key centres (kt, ky, kx) of the reference tape, as float64."""
        import torch

        rows = self.sims.shape[0]
        t, nh, nw = self._grid
        s0 = self.cfg.stride0
        r = torch.arange(rows, device=self.sims.device)
        qx = (r % nw) * s0
        qy = ((r // nw) % nh) * s0
        qt = r // (nw * nh)
        base = torch.stack([qt, qy, qx], -1).double()[:, None, :]
        return base + self.offsets.double()


def shifted_nls_forward(q, k, fflow, bflow, cfg: SearchConfig, mode: int = MODE_FUSED,
                        want_chains: bool = True, want_weights: bool = False,
                        ctx: Optional[Context] = None, check: bool = True, out=None,
                        frames=None) -> SearchResult:
    """snls::shifted_nls_forward (search.hpp:126-128). fflow/bflow None => nls_forward.
    `frames=(t0, t1)` searches only the query rows of frames [t0, t1) (frame sharding)."""
    import torch

    ctx = ctx or context(q.device.index)
    t, h, w, f = q.shape
    t0, t1 = frames if frames is not None else (0, t)
    if tuple(k.shape) != tuple(q.shape):
        raise DomainError("search: query and key shapes differ")
    if fflow is not None and (tuple(fflow.shape) != (t, h, w, 2) or tuple(bflow.shape) != (t, h, w, 2)):
        raise DomainError("search: flow shape does not match the video")
    c = _cfg(cfg)
    _raise(lib().snls_validate_config(C.byref(c)))
    rows = (t1 - t0) * ((h - 1) // cfg.stride0 + 1) * ((w - 1) // cfg.stride0 + 1)
    if out is None:
        sims = torch.empty((rows, cfg.topl), device=q.device, dtype=torch.float32)
        offs = torch.empty((rows, cfg.topl, 3), device=q.device, dtype=torch.float32)
        chains = (torch.empty((rows, cfg.topl, cfg.chain_stride(), 6), device=q.device,
                              dtype=torch.float32) if want_chains and cfg.wt > 1 else None)
        weights = (torch.empty((rows, cfg.topl), device=q.device, dtype=torch.float32)
                   if want_weights else None)
    else:
        sims, offs, chains, weights = out
    _raise(lib().snls_search_fwd_frames(ctx.h, C.byref(c), _dims(q), int(t0), int(t1), _ptr(q),
                                        _ptr(k), _ptr(fflow), _ptr(bflow), int(mode), _ptr(sims),
                                        _ptr(offs), _ptr(chains), _ptr(weights)))
    if check:
        ctx.sync_check()
    res = SearchResult(sims, offs, chains, weights, cfg)
    res._grid = (t1 - t0, (h - 1) // cfg.stride0 + 1, (w - 1) // cfg.stride0 + 1)
    return res


def nls_forward(q, k, cfg: SearchConfig, **kw) -> SearchResult:
    """snls::nls_forward (search.hpp:131-132): both flows identically zero."""
    return shifted_nls_forward(q, k, None, None, cfg, **kw)


def search_grid(q, k, fflow, bflow, cfg: SearchConfig, ctx=None):
    """Materialised pre-selection grid (full_grid_forward, search.cpp:351-376)."""
    import torch

    ctx = ctx or context(q.device.index)
    t, h, w, f = q.shape
    c = _cfg(cfg)
    rows = t * ((h - 1) // cfg.stride0 + 1) * ((w - 1) // cfg.stride0 + 1)
    n = cfg.window_slots()
    grid = torch.empty((rows, n), device=q.device, dtype=torch.float32)
    goff = torch.empty((rows, n, 3), device=q.device, dtype=torch.float32)
    _raise(lib().snls_search_grid(ctx.h, C.byref(c), _dims(q), _ptr(q), _ptr(k), _ptr(fflow),
                                  _ptr(bflow), _ptr(grid), _ptr(goff)))
    ctx.sync_check()
    return grid, goff


def top_l(full, full_offsets, topl: int, ctx=None):
    """snls::top_l (search.hpp:137-138)."""
    import torch

    ctx = ctx or context(full.device.index)
    rows, cols = full.shape
    if tuple(full_offsets.shape) != (rows, cols, 3):
        raise DomainError("top_l: similarity and offset shapes disagree")
    sel = torch.empty((rows, max(topl, 1)), device=full.device, dtype=torch.float32)
    soff = torch.empty((rows, max(topl, 1), 3), device=full.device, dtype=torch.float32)
    _raise(lib().snls_topl(ctx.h, rows, cols, _ptr(full), _ptr(full_offsets), int(topl),
                           _ptr(sel), _ptr(soff)))
    ctx.sync_check()
    return sel, soff


def replay_similarities(res: SearchResult, q, k, ctx=None, centers=None, plan: str = "auto"):
    """snls::replay_similarities (search.hpp:157-158).  With the fp64 tape `centers`
    (search_tape64) through the search plan's own arithmetic -- bitwise equal to that plan's
    forward (snls_replay64; plan 'auto' = the one the forward takes); without, from the fp32
    device tape (snls_replay, fp32 tolerance)."""
    import torch

    ctx = ctx or context(q.device.index)
    c = _cfg(res.cfg)
    sims = torch.empty_like(res.sims)
    if centers is not None:
        t = q.shape[0]
        _raise(lib().snls_replay64(ctx.h, C.byref(c), _dims(q), 0, t, _ptr(q), _ptr(k), _ptr(centers),
                                   {"auto": -1, "generic": 0, "tiled": 1, "stream": 2}[plan], _ptr(sims)))
    else:
        _raise(lib().snls_replay(ctx.h, C.byref(c), _dims(q), _ptr(q), _ptr(k), _ptr(res.offsets),
                                 _ptr(sims)))
    ctx.sync_check()
    return sims


def search_tape64(res: SearchResult, fflow, bflow, ctx=None, frames=None, check=True, out=None):
    """The reference's fp64 SearchTape (search.hpp:89-110) of a device result: absolute
    centres rows x L x 3 and (wt > 1) absolute chain links rows x L x (wt-1) x 6, float64."""
    import torch

    ctx = ctx or context(res.sims.device.index)
    cfg = res.cfg
    c = _cfg(cfg)
    if fflow is None:
        raise SnlsError("search_tape64: pass the flows (zeros for nls_forward)")
    t, h, w = fflow.shape[:3]
    t0, t1 = frames if frames is not None else (0, t)
    rows, L = res.sims.shape
    if out is None:
        cen = torch.empty((rows, L, 3), device=res.sims.device, dtype=torch.float64)
        ch = (torch.empty((rows, L, cfg.chain_stride(), 6), device=res.sims.device, dtype=torch.float64)
              if cfg.wt > 1 else None)
    else:
        cen, ch = out
    _raise(lib().snls_search_tape64(ctx.h, C.byref(c), _Dims(t, h, w, 1), int(t0), int(t1),
                                    _ptr(fflow), _ptr(bflow), _ptr(res.offsets), _ptr(cen), _ptr(ch)))
    if check:
        ctx.sync_check()
    return cen, ch


def shifted_nls_backward(grad_sims, res: SearchResult, q, k, ctx=None, check=True, frames=None,
                         deterministic=False, tape64=None):
    """snls::shifted_nls_backward (search.hpp:151-153) -> (dq, dk, dfflow, dbflow).
    `frames=(t0, t1)`: the tape holds the rows of query frames [t0, t1) only (frame
    sharding); the gradients still cover every frame of q / k.  `deterministic`: the
    reference's default mode (bitwise reproducible, search.cpp:687-696).  `tape64`:
    (centers, chains64) -- the reference's fp64 tape (search_tape64) instead of the device
    tape."""
    import torch

    ctx = ctx or context(q.device.index)
    c = _cfg(res.cfg)
    t, h, w, f = q.shape
    t0, t1 = frames if frames is not None else (0, t)
    if tuple(grad_sims.shape) != tuple(res.sims.shape):
        raise DomainError("shifted_nls_backward: gradient shape does not match the tape")
    dq = torch.empty_like(q)
    dk = torch.empty_like(q)
    dff = torch.empty((t, h, w, 2), device=q.device, dtype=torch.float32)
    dbf = torch.empty_like(dff)
    cen, ch64 = tape64 if tape64 is not None else (None, None)
    _raise(lib().snls_search_bwd_ex(ctx.h, C.byref(c), _dims(q), int(t0), int(t1), _ptr(grad_sims),
                                    None if cen is not None else _ptr(res.offsets),
                                    None if cen is not None else _ptr(res.chains), _ptr(cen),
                                    _ptr(ch64), _ptr(q), _ptr(k), _ptr(dq), _ptr(dk), _ptr(dff),
                                    _ptr(dbf), 1 if deterministic else 0))
    if check:
        ctx.sync_check()
    return dq, dk, dff, dbf


def train_backward(grad_sims, grad_out, counts, res: SearchResult, q, k, v, ctx=None, check=True,
                   deterministic=False, tape64=None):
    """The backward of search -> softmax weights -> wpsum in one call (snls_train_bwd):
    returns (dq, dk, dv, dfflow, dbflow, dweights) as shifted_nls_backward + wpsum_backward;
    when v is k one fused kernel serves both."""
    import torch

    ctx = ctx or context(q.device.index)
    c = _cfg(res.cfg)
    t, h, w, f = q.shape
    dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(v)
    dff = torch.empty((t, h, w, 2), device=q.device, dtype=torch.float32)
    dbf = torch.empty_like(dff)
    dw = torch.empty_like(res.weights)
    cen, ch64 = tape64 if tape64 is not None else (None, None)
    _raise(lib().snls_train_bwd(ctx.h, C.byref(c), _dims(q), _ptr(grad_sims), _ptr(grad_out), _ptr(counts),
                                _ptr(res.offsets), _ptr(res.chains), _ptr(cen), _ptr(ch64), _ptr(q), _ptr(k),
                                _ptr(v), _ptr(res.weights), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(dw), _ptr(dff),
                                _ptr(dbf), 1 if deterministic else 0))
    if check:
        ctx.sync_check()
    return dq, dk, dv, dff, dbf, dw


def softmax_rows(sims, beta: float, ctx=None, check=True):
    """snls::softmax_rows (aggregate.hpp:22)."""
    import torch

    ctx = ctx or context(sims.device.index)
    rows, l = sims.shape
    w = torch.empty_like(sims)
    _raise(lib().snls_softmax_rows(ctx.h, rows, l, float(beta), _ptr(sims), _ptr(w)))
    if check:
        ctx.sync_check()
    return w


def _agg_shape_checks(v, weights, offsets, cfg, frames=None):
    t, h, w, f = v.shape
    t0, t1 = frames if frames is not None else (0, t)
    rows = (t1 - t0) * ((h - 1) // cfg.stride0 + 1) * ((w - 1) // cfg.stride0 + 1)
    validate(cfg)
    if not cfg.hole_free():
        raise ConfigError("aggregate: (ps-1)/2 < stride0 is required for hole-free output")
    if weights.shape[0] != rows or offsets.shape[0] != rows:
        raise DomainError("aggregate: weight/offset rows do not match the query grid")
    if weights.shape[1] != offsets.shape[1] or weights.shape[1] != cfg.topl:
        raise DomainError("aggregate: weight/offset L does not match the config")


def wpsum(v, weights, offsets, cfg: SearchConfig, ctx=None, check=True, out=None, frames=None):
    """snls::wpsum (aggregate.hpp:53-54) -> (video, counts).  `frames=(t0, t1)` aggregates
    only the output frames [t0, t1) from those frames' query rows (frame sharding)."""
    import torch

    ctx = ctx or context(v.device.index)
    _agg_shape_checks(v, weights, offsets, cfg, frames)
    c = _cfg(cfg)
    t, h, w, f = v.shape
    t0, t1 = frames if frames is not None else (0, t)
    if out is None:
        o = torch.empty((t1 - t0, h, w, f), device=v.device, dtype=torch.float32)
        counts = torch.empty((t1 - t0, h, w), device=v.device, dtype=torch.int32)
    else:
        o, counts = out
    _raise(lib().snls_wpsum_fwd_frames(ctx.h, C.byref(c), _dims(v), int(t0), int(t1), _ptr(v),
                                       _ptr(weights), _ptr(offsets), _ptr(o), _ptr(counts)))
    if check:
        ctx.sync_check()
    return o, counts


def gather_stack(v, weights, offsets, cfg: SearchConfig, ctx=None, check=True):
    """snls::gather_stack (aggregate.hpp:71-73) -> L x T x H x W x F."""
    import torch

    ctx = ctx or context(v.device.index)
    _agg_shape_checks(v, weights, offsets, cfg)
    c = _cfg(cfg)
    out = torch.empty((cfg.topl, *v.shape), device=v.device, dtype=torch.float32)
    _raise(lib().snls_gather_stack(ctx.h, C.byref(c), _dims(v), _ptr(v), _ptr(weights),
                                   _ptr(offsets), _ptr(out)))
    if check:
        ctx.sync_check()
    return out


def wpsum_backward(grad_out, counts, v, weights, offsets, cfg: SearchConfig, ctx=None, check=True,
                   frames=None, deterministic=False):
    """snls::wpsum_backward (aggregate.hpp:83-85) -> (dv, dweights).  `frames=(t0, t1)`:
    grad_out / counts / weights / offsets hold output frames [t0, t1) only; dv covers v.
    `deterministic`: the reference's ExecPolicy::deterministic (aggregate.cpp:439-450) --
    bitwise identical results run to run (int64 fixed-point accumulation of dV)."""
    import torch

    ctx = ctx or context(v.device.index)
    t0, t1 = frames if frames is not None else (0, v.shape[0])
    if tuple(grad_out.shape) != (t1 - t0,) + tuple(v.shape[1:]):
        raise DomainError("wpsum_backward: gradient shape does not match the tape")
    c = _cfg(cfg)
    dv = torch.empty_like(v)
    dw = torch.empty_like(weights)
    _raise(lib().snls_wpsum_bwd_ex(ctx.h, C.byref(c), _dims(v), int(t0), int(t1), _ptr(grad_out),
                                   _ptr(counts), _ptr(v), _ptr(weights), _ptr(offsets), _ptr(dv),
                                   _ptr(dw), 1 if deterministic else 0))
    if check:
        ctx.sync_check()
    return dv, dw


# ---------------------------------------------------------------------------------------
class Pipeline:
    """Host-buffer search + fused softmax + wpsum over a clip (snls_pipeline_*, see
    include/snls_cuda.h): frame-chunked kernels overlapped with the H2D input and D2H result
    copies.  Arguments of run() are HOST tensors/arrays (torch CPU tensors -- pinned for
    overlap -- or numpy arrays); q, k, v may be the same buffer (copied once)."""

    def __init__(self, cfg: SearchConfig, dims, chunk_frames: int = 1, ctx: Optional[Context] = None):
        self.ctx = ctx or context()
        self.cfg = cfg
        self.dims = tuple(int(x) for x in dims)
        self._c = _cfg(cfg)
        h = VOIDP()
        _raise(lib().snls_pipeline_create(self.ctx.h, C.byref(self._c), _Dims(*self.dims),
                                          int(chunk_frames), C.byref(h)))
        self.h = h

    @staticmethod
    def _hp(x):
        if x is None:
            return None
        if hasattr(x, "data_ptr"):
            if x.is_cuda or not x.is_contiguous():
                raise SnlsError("snls pipeline: host buffers must be contiguous CPU tensors")
            return VOIDP(x.data_ptr())
        if not x.flags["C_CONTIGUOUS"]:
            raise SnlsError("snls pipeline: host buffers must be C-contiguous")
        return VOIDP(x.ctypes.data)

    def run(self, q, k, v, fflow, bflow, sims=None, offsets=None, weights=None, out=None,
            counts=None):
        hp = self._hp
        _raise(lib().snls_pipeline_run(self.h, hp(q), hp(k), hp(v), hp(fflow), hp(bflow),
                                       hp(sims), hp(offsets), hp(weights), hp(out), hp(counts)))

    def submit(self, q, k, v, fflow, bflow, sims=None, offsets=None, weights=None, out=None,
               counts=None):
        """Streaming form: enqueue a clip (at most three in flight); the buffers must stay
        alive and untouched until the matching wait()."""
        hp = self._hp
        _raise(lib().snls_pipeline_submit(self.h, hp(q), hp(k), hp(v), hp(fflow), hp(bflow),
                                          hp(sims), hp(offsets), hp(weights), hp(out), hp(counts)))

    def wait(self):
        """Block until the oldest submitted clip's results are in host memory."""
        _raise(lib().snls_pipeline_wait(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().snls_pipeline_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def host_register(buf) -> None:
    """Pin a host numpy array / CPU tensor in place (cudaHostRegister)."""
    ptr = buf.data_ptr() if hasattr(buf, "data_ptr") else buf.ctypes.data
    n = buf.numel() * buf.element_size() if hasattr(buf, "numel") else buf.nbytes
    _raise(lib().snls_host_register(VOIDP(ptr), n))


# ---------------------------------------------------------------------------------------
# frame alignment: flow.cpp:114-175, tensor.cpp:79-99, harness.cpp:72-154
FLOW_ZERO, FLOW_PROVIDED, FLOW_BLOCK_MATCHING = 0, 1, 2


def block_match(a, b, block: int = 9, radius: int = 8, ctx=None):
    """estimate_flow_block_matching for every frame pair a[t] -> b[t] (torch CUDA T x H x W x F)
    -> flow T x H x W x 2."""
    import torch

    ctx = ctx or context(a.device.index)
    if tuple(a.shape) != tuple(b.shape):
        raise DomainError("estimate_flow_block_matching: shape mismatch")
    t, h, w, f = a.shape
    flow = torch.empty((t, h, w, 2), device=a.device, dtype=torch.float32)
    _raise(lib().snls_block_match(ctx.h, _Dims(t, h, w, f), _ptr(a), _ptr(b), int(block), int(radius),
                                  _ptr(flow)))
    return flow


def psnr_frames(a, b, peak: float = 255.0, ctx=None):
    """psnr (tensor.cpp:79-90) per frame -> list of floats."""
    ctx = ctx or context(a.device.index)
    if tuple(a.shape) != tuple(b.shape):
        raise DomainError("psnr: shape mismatch")
    t = a.shape[0]
    out = (C.c_double * t)()
    _raise(lib().snls_psnr_frames(ctx.h, _dims(a), _ptr(a), _ptr(b), float(peak), out))
    return list(out)


def add_gaussian_noise(v, sigma: float, seed: int):
    """add_gaussian_noise (tensor.cpp:92-99) on a float32 numpy array (host)."""
    import numpy as np

    v = np.ascontiguousarray(v, dtype=np.float32)
    out = np.empty_like(v)
    _raise(lib().snls_gaussian_noise_f32(C.c_uint64(seed), float(sigma), v.size, v.ctypes.data,
                                         out.ctypes.data))
    return out


def align_frames(clean, cfg: SearchConfig, flow_source: int = FLOW_ZERO, provided_flow=None,
                 sigma: float = 0.0, seed: int = 0, bm_block: int = 9, bm_radius: int = 8, ctx=None):
    """snls::align_frames (harness.hpp:61-62) over a HOST float32 clip T x H x W x F ->
    dict(aligned, top1_offsets, used_flow, frame_psnr, mean_psnr)."""
    import numpy as np

    ctx = ctx or context()
    clean = np.ascontiguousarray(clean, dtype=np.float32)
    t, h, w, f = clean.shape
    c = _cfg(cfg)
    pairs = max(t - 1, 0)
    nq = ((h - 1) // cfg.stride0 + 1) * ((w - 1) // cfg.stride0 + 1)
    aligned = np.zeros((pairs, h, w, f), np.float32)
    offs = np.zeros((pairs * nq, 3), np.float32)
    used = np.zeros((pairs, h, w, 2), np.float32)
    ps = np.zeros(pairs, np.float64)
    prov = None
    if provided_flow is not None:
        prov = np.ascontiguousarray(provided_flow, dtype=np.float32)
        if prov.shape[1:3] != (h, w) or prov.shape[0] < pairs:
            raise DomainError("align_frames: provided flow does not cover every frame pair")
    _raise(lib().snls_align_frames(ctx.h, C.byref(c), _Dims(t, h, w, f), clean.ctypes.data,
                                   float(sigma), C.c_uint64(seed), int(flow_source),
                                   None if prov is None else prov.ctypes.data, int(bm_block),
                                   int(bm_radius), aligned.ctypes.data, offs.ctypes.data,
                                   used.ctypes.data, ps.ctypes.data))
    return {"aligned": aligned, "top1_offsets": offs, "used_flow": used, "frame_psnr": ps,
            "mean_psnr": float(ps.mean()) if pairs else float("nan")}


# ---------------------------------------------------------------------------------------
# on-disk formats: .stnt (video_io.cpp:52-117), .flo (flow.cpp:53-112)
def read_raw(path: str):
    """load_raw -> float32 numpy T x H x W x F (and the file's element width)."""
    import numpy as np

    d, wd = _Dims(), C.c_int()
    _raise(lib().snls_raw_info(path.encode(), C.byref(d), C.byref(wd)))
    out = np.empty((d.t, d.h, d.w, d.f), np.float32)
    _raise(lib().snls_raw_read(path.encode(), out.ctypes.data, out.size))
    return out


def write_raw(path: str, v, width: int = 4) -> None:
    """save_raw from a float32 array T x H x W x F (width 4: f32 payload, 8: f64)."""
    import numpy as np

    v = np.ascontiguousarray(v, dtype=np.float32)
    _raise(lib().snls_raw_write(path.encode(), _Dims(*v.shape), v.ctypes.data, int(width)))


def read_flo(path: str):
    """read_flo -> float32 numpy H x W x 2 holding (dy, dx)."""
    import numpy as np

    h, w = C.c_int(), C.c_int()
    _raise(lib().snls_flo_read(path.encode(), C.byref(h), C.byref(w), None))
    out = np.empty((h.value, w.value, 2), np.float32)
    _raise(lib().snls_flo_read(path.encode(), C.byref(h), C.byref(w), out.ctypes.data))
    return out


def write_flo(path: str, flow) -> None:
    """write_flo of one H x W x 2 (dy, dx) field."""
    import numpy as np

    flow = np.ascontiguousarray(flow, dtype=np.float32)
    _raise(lib().snls_flo_write(path.encode(), flow.shape[0], flow.shape[1], flow.ctypes.data))
