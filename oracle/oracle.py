"""TEST INFRASTRUCTURE ONLY -- ctypes front end for the two CPU checkers.

* ``Checker("port")``      -> oracle/liboracle_snls.so, the plain-C restatement (snls_oracle.c)
* ``Checker("reference")`` -> oracle/_ref/libsnls_ref.so, the reference's own sources compiled
  unmodified (oracle/Makefile) behind the shim ref_capi.cpp

Both expose the same methods over numpy float64 arrays so a test can run one against the
other.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import this
module; the product (paper_2309_16849_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "liboracle_snls.so")
REF_LIB = os.path.join(HERE, "_ref", "libsnls_ref.so")


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.kind = {1: "ConfigError", 2: "DomainError"}.get(code, "Error")


@dataclass
class Cfg:
    """Mirror of snls::SearchConfig (search.hpp:17-26); metric 'ip' or 'l2'."""

    ws: int = 9
    wt: int = 0
    ps: int = 1
    stride0: int = 1
    stride1: float = 1.0
    topl: int = 1
    metric: str = "l2"
    softmax_scale: float = 1.0

    def window_slots(self) -> int:
        return (2 * self.wt + 1) * self.ws * self.ws

    def hole_free(self) -> bool:
        return (self.ps - 1) // 2 < self.stride0


class _CCfg(C.Structure):
    _fields_ = [("ws", C.c_int), ("wt", C.c_int), ("ps", C.c_int), ("stride0", C.c_int),
                ("stride1", C.c_double), ("topl", C.c_int), ("metric", C.c_int),
                ("softmax_scale", C.c_double)]


def _ccfg(c: Cfg) -> _CCfg:
    return _CCfg(c.ws, c.wt, c.ps, c.stride0, float(c.stride1), c.topl,
                 0 if c.metric == "ip" else 1, float(c.softmax_scale))


def query_grid(t: int, h: int, w: int, stride0: int):
    nh = (h - 1) // stride0 + 1
    nw = (w - 1) // stride0 + 1
    return t * nh * nw, nh, nw


def build(quiet: bool = True) -> None:
    """Compile both checkers (the reference one only where /root/reference exists)."""
    subprocess.run(["make", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


_P = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def _d(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _iptr(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int32))


class Checker:
    def __init__(self, which: str = "port"):
        self.which = which
        path = PORT_LIB if which == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self.pre = "oracle_" if which == "port" else "ref_"
        getattr(self.lib, self.pre + "last_error").restype = C.c_char_p
        getattr(self.lib, self.pre + "uniform_bits").restype = C.c_uint64
        getattr(self.lib, self.pre + "uniform_bits").argtypes = [C.c_uint64, C.c_int64]
        getattr(self.lib, self.pre + "uniform_fill").argtypes = [C.c_uint64, C.c_double, C.c_double,
                                                        C.c_int64, C.POINTER(C.c_double)]

    def _fn(self, name):
        return getattr(self.lib, self.pre + name)

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self._fn("last_error")().decode())

    # ---- rng.hpp / tensor.cpp primitives ----
    def uniform(self, seed: int, lo: float, hi: float, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self._fn("uniform_fill")(C.c_uint64(seed), lo, hi, n, _ptr(out))
        return out

    def uniform_bits(self, seed: int, skip: int = 0) -> int:
        return int(self._fn("uniform_bits")(C.c_uint64(seed), skip))

    def reflect_index(self, i: int, n: int) -> int:
        return int(self._fn("reflect_index")(i, n))

    def bilinear_taps(self, h, w, y, x):
        idx = np.zeros(4, np.int32)
        wts = np.zeros(6, np.float64)
        self._fn("bilinear_taps")(h, w, C.c_double(y), C.c_double(x), _iptr(idx), _ptr(wts))
        return idx, wts

    def validate(self, cfg: Cfg):
        c = _ccfg(cfg)
        self._check(self._fn("validate")(C.byref(c)))

    def accumulate_shift(self, ff, bf, qt, qy, qx, dt, links=False):
        ff, bf = _d(ff), _d(bf)
        t, h, w = ff.shape[:3]
        dy, dx = C.c_double(), C.c_double()
        lk = np.zeros(max(abs(dt) - 1, 1) * 6) if links else None
        self._check(self._fn("accumulate_shift")(t, h, w, _ptr(ff), _ptr(bf), qt, qy, qx, dt,
                                                 C.byref(dy), C.byref(dx), _ptr(lk)))
        return (dy.value, dx.value, lk) if links else (dy.value, dx.value)

    # ---- search.hpp ----
    def search_fwd(self, q, k, ff, bf, cfg: Cfg, mode: int = 0, threads: int = 0):
        q, k, ff, bf = _d(q), _d(k), _d(ff), _d(bf)
        t, h, w, f = q.shape
        rows, _, _ = query_grid(t, h, w, cfg.stride0)
        L = cfg.topl
        cs = max(cfg.wt - 1, 0)
        sims = np.zeros((rows, L))
        offs = np.zeros((rows, L, 3))
        cent = np.zeros((rows, L, 3))
        chains = np.zeros((rows, L, cs, 6))
        c = _ccfg(cfg)
        if self.which == "port":
            rc = self._fn("search_fwd")(t, h, w, f, _ptr(q), _ptr(k), _ptr(ff), _ptr(bf),
                                        C.byref(c), _ptr(sims), _ptr(offs), _ptr(cent),
                                        _ptr(chains))
        else:
            rc = self._fn("search_fwd")(t, h, w, f, _ptr(q), _ptr(k), _ptr(ff), _ptr(bf),
                                        C.byref(c), mode, threads, _ptr(sims), _ptr(offs),
                                        _ptr(cent), _ptr(chains))
        self._check(rc)
        return {"sims": sims, "offsets": offs, "centers": cent, "chains": chains}

    def serial_search_fwd(self, q, k, ff, bf, cfg: Cfg):
        """snls::reference::shifted_nls_forward (reference.cpp:18-109); reference lib only."""
        q, k, ff, bf = _d(q), _d(k), _d(ff), _d(bf)
        t, h, w, f = q.shape
        rows, _, _ = query_grid(t, h, w, cfg.stride0)
        L, cs = cfg.topl, max(cfg.wt - 1, 0)
        sims, offs = np.zeros((rows, L)), np.zeros((rows, L, 3))
        cent, chains = np.zeros((rows, L, 3)), np.zeros((rows, L, cs, 6))
        c = _ccfg(cfg)
        self._check(self.lib.ref_serial_search_fwd(t, h, w, f, _ptr(q), _ptr(k), _ptr(ff),
                                                   _ptr(bf), C.byref(c), _ptr(sims), _ptr(offs),
                                                   _ptr(cent), _ptr(chains)))
        return {"sims": sims, "offsets": offs, "centers": cent, "chains": chains}

    def search_full_grid(self, q, k, ff, bf, cfg: Cfg):
        """Pre-selection window grid (port only; search.cpp:329-376)."""
        q, k, ff, bf = _d(q), _d(k), _d(ff), _d(bf)
        t, h, w, f = q.shape
        rows, _, _ = query_grid(t, h, w, cfg.stride0)
        n = cfg.window_slots()
        grid, goff = np.zeros((rows, n)), np.zeros((rows, n, 3))
        c = _ccfg(cfg)
        self._check(self.lib.oracle_search_full_grid(t, h, w, f, _ptr(q), _ptr(k), _ptr(ff),
                                                     _ptr(bf), C.byref(c), _ptr(grid),
                                                     _ptr(goff)))
        return grid, goff

    def top_l(self, full, full_offsets, topl: int):
        full, full_offsets = _d(full), _d(full_offsets)
        rows, cols = full.shape
        sel, soff = np.zeros((rows, topl)), np.zeros((rows, topl, 3))
        self._check(self._fn("top_l")(C.c_int64(rows), cols, _ptr(full), _ptr(full_offsets),
                                      topl, _ptr(sel), _ptr(soff)))
        return sel, soff

    def replay(self, q, k, cfg: Cfg, centers, chains=None):
        q, k, centers = _d(q), _d(k), _d(centers)
        t, h, w, f = q.shape
        rows, _, _ = query_grid(t, h, w, cfg.stride0)
        sims = np.zeros((rows, cfg.topl))
        c = _ccfg(cfg)
        if self.which == "port":
            rc = self._fn("replay")(t, h, w, f, _ptr(q), _ptr(k), C.byref(c), _ptr(centers),
                                    _ptr(sims))
        else:
            ch = _d(chains) if chains is not None else np.zeros(1)
            rc = self._fn("replay")(t, h, w, f, _ptr(q), _ptr(k), C.byref(c), _ptr(centers),
                                    _ptr(ch), _ptr(sims))
        self._check(rc)
        return sims

    def search_bwd(self, q, k, cfg: Cfg, centers, chains, grad_sims, deterministic=True,
                   threads=0):
        q, k, centers, grad_sims = _d(q), _d(k), _d(centers), _d(grad_sims)
        chains = _d(chains) if chains is not None and chains.size else np.zeros(1)
        t, h, w, f = q.shape
        dq, dk = np.zeros_like(q), np.zeros_like(q)
        dff, dbf = np.zeros((t, h, w, 2)), np.zeros((t, h, w, 2))
        c = _ccfg(cfg)
        if self.which == "port":
            rc = self._fn("search_bwd")(t, h, w, f, _ptr(q), _ptr(k), C.byref(c), _ptr(centers),
                                        _ptr(chains), _ptr(grad_sims), _ptr(dq), _ptr(dk),
                                        _ptr(dff), _ptr(dbf))
        else:
            rc = self._fn("search_bwd")(t, h, w, f, _ptr(q), _ptr(k), C.byref(c), _ptr(centers),
                                        _ptr(chains), _ptr(grad_sims), int(deterministic),
                                        threads, _ptr(dq), _ptr(dk), _ptr(dff), _ptr(dbf))
        self._check(rc)
        return {"dq": dq, "dk": dk, "dfflow": dff, "dbflow": dbf}

    # ---- aggregate.hpp ----
    def softmax_rows(self, sims, beta: float):
        sims = _d(sims)
        rows, l = sims.shape
        out = np.zeros_like(sims)
        self._check(self._fn("softmax_rows")(C.c_int64(rows), l, _ptr(sims), C.c_double(beta),
                                             _ptr(out)))
        return out

    def wpsum(self, v, weights, offsets, cfg: Cfg, deterministic=True, threads=0,
              serial_reference=False):
        v, weights, offsets = _d(v), _d(weights), _d(offsets)
        t, h, w, f = v.shape
        rows, l = weights.shape
        out = np.zeros_like(v)
        counts = np.zeros((t, h, w), np.int32)
        c = _ccfg(cfg)
        if self.which == "port":
            rc = self._fn("wpsum")(t, h, w, f, _ptr(v), C.c_int64(rows), l, _ptr(weights),
                                   _ptr(offsets), C.byref(c), _ptr(out), _iptr(counts))
        else:
            rc = self._fn("wpsum")(t, h, w, f, _ptr(v), C.c_int64(rows), l, _ptr(weights),
                                   _ptr(offsets), C.byref(c), int(deterministic), threads,
                                   int(serial_reference), _ptr(out), _iptr(counts))
        self._check(rc)
        return out, counts

    def gather_stack(self, v, weights, offsets, cfg: Cfg, threads=0, serial_reference=False):
        v, weights, offsets = _d(v), _d(weights), _d(offsets)
        t, h, w, f = v.shape
        rows, l = weights.shape
        out = np.zeros((l, t, h, w, f))
        c = _ccfg(cfg)
        if self.which == "port":
            rc = self._fn("gather_stack")(t, h, w, f, _ptr(v), C.c_int64(rows), l, _ptr(weights),
                                          _ptr(offsets), C.byref(c), _ptr(out))
        else:
            rc = self._fn("gather_stack")(t, h, w, f, _ptr(v), C.c_int64(rows), l, _ptr(weights),
                                          _ptr(offsets), C.byref(c), threads,
                                          int(serial_reference), _ptr(out))
        self._check(rc)
        return out

    def wpsum_bwd(self, grad_out, counts, v, weights, offsets, cfg: Cfg, deterministic=True,
                  threads=0):
        grad_out, v, weights, offsets = _d(grad_out), _d(v), _d(weights), _d(offsets)
        counts = np.ascontiguousarray(counts, dtype=np.int32)
        t, h, w, f = v.shape
        rows, l = weights.shape
        dv, dw = np.zeros_like(v), np.zeros_like(weights)
        c = _ccfg(cfg)
        if self.which == "port":
            rc = self._fn("wpsum_bwd")(t, h, w, f, _ptr(grad_out), _iptr(counts), _ptr(v),
                                       C.c_int64(rows), l, _ptr(weights), _ptr(offsets),
                                       C.byref(c), _ptr(dv), _ptr(dw))
        else:
            rc = self._fn("wpsum_bwd")(t, h, w, f, _ptr(grad_out), _iptr(counts), _ptr(v),
                                       C.c_int64(rows), l, _ptr(weights), _ptr(offsets),
                                       C.byref(c), int(deterministic), threads, _ptr(dv),
                                       _ptr(dw))
        self._check(rc)
        return dv, dw


    # ---- frame alignment pieces (flow.cpp:114-175, tensor.cpp:79-99, harness.cpp:72-154) ----
    def block_match(self, a, b, block: int, radius: int):
        """a, b: single frames h x w x f -> flow h x w x 2 (estimate_flow_block_matching)."""
        a, b = _d(a), _d(b)
        h, w, f = a.shape
        flow = np.zeros((h, w, 2))
        self._check(self._fn("block_match")(h, w, f, _ptr(a), _ptr(b), block, radius, _ptr(flow)))
        return flow

    def psnr(self, a, b, peak: float = 255.0) -> float:
        a, b = _d(a), _d(b)
        out = C.c_double()
        if self.which == "port":
            self._check(self._fn("psnr")(C.c_int64(a.size), _ptr(a), _ptr(b), C.c_double(peak),
                                         C.byref(out)))
        else:
            t, h, w, f = a.shape if a.ndim == 4 else (1,) + a.shape
            self._check(self._fn("psnr")(t, h, w, f, _ptr(a), _ptr(b), C.c_double(peak), C.byref(out)))
        return out.value

    def add_gaussian_noise(self, v, sigma: float, seed: int):
        """tensor.cpp:92-99: v + sigma * GaussianStream(seed), element order."""
        v = _d(v)
        if self.which == "port":
            g = np.empty(v.size)
            self.lib.oracle_gaussian_fill.argtypes = [C.c_uint64, C.c_int64, C.POINTER(C.c_double)]
            self.lib.oracle_gaussian_fill(C.c_uint64(seed), v.size, _ptr(g))
            return v + sigma * g.reshape(v.shape) if sigma != 0.0 else v.copy()
        out = np.empty_like(v)
        t, h, w, f = v.shape
        self._check(self._fn("add_gaussian_noise")(t, h, w, f, _ptr(v), C.c_double(sigma),
                                                   C.c_uint64(seed), _ptr(out)))
        return out

    def align_frames(self, clean, cfg: Cfg, source: int = 0, provided=None, sigma: float = 0.0,
                     seed: int = 0, bm_block: int = 9, bm_radius: int = 8, noisy=None):
        """harness.cpp:72-154.  port: the restated pieces composed in the reference's order
        (noise, per-pair flow, per-pair search / softmax / wpsum / psnr); `noisy` overrides
        the noise step (e.g. fp32-rounded noisy frames).  reference: snls::align_frames."""
        clean = _d(clean)
        t, h, w, f = clean.shape
        if self.which != "port":
            nq = ((h - 1) // cfg.stride0 + 1) * ((w - 1) // cfg.stride0 + 1)
            aligned = np.zeros((t - 1, h, w, f))
            offs = np.zeros(((t - 1) * nq, 3))
            used = np.zeros((t - 1, h, w, 2))
            ps = np.zeros(t - 1)
            prov = _d(provided) if provided is not None else np.zeros(1)
            c = _ccfg(cfg)
            self._check(self._fn("align_frames")(t, h, w, f, _ptr(clean), C.byref(c), source,
                                                 _ptr(prov), C.c_double(sigma), C.c_uint64(seed),
                                                 bm_block, bm_radius, _ptr(aligned), _ptr(offs),
                                                 _ptr(used), _ptr(ps)))
            return {"aligned": aligned, "offsets": offs, "used_flow": used, "psnr": ps}
        if noisy is None:
            noisy = self.add_gaussian_noise(clean, sigma, seed) if sigma > 0 else clean
        used = np.zeros((t - 1, h, w, 2))
        for ti in range(t - 1):
            if source == 1:
                used[ti] = provided[ti]
            elif source == 2:
                used[ti] = self.block_match(noisy[ti], noisy[ti + 1], bm_block, bm_radius)
        zero_b = np.zeros((1, h, w, 2))
        aligned, offs, ps = [], [], []
        for ti in range(t - 1):
            r = self.search_fwd(noisy[ti:ti + 1], noisy[ti + 1:ti + 2], used[ti:ti + 1], zero_b, cfg)
            wts = self.softmax_rows(r["sims"], cfg.softmax_scale)
            out, _ = self.wpsum(clean[ti + 1:ti + 2], wts, r["offsets"], cfg)
            aligned.append(out[0])
            offs.append(r["offsets"].reshape(-1, 3))
            ps.append(self.psnr(out[0], clean[ti]))
        return {"aligned": np.stack(aligned), "offsets": np.concatenate(offs), "used_flow": used,
                "psnr": np.array(ps)}


def have_reference() -> bool:
    return os.path.exists(REF_LIB)
