"""Python mirror of the reference's stepping API over the laxol_b200 C-ABI.

Names and argument meaning follow the reference (`laxol`, /root/reference/proj):
``build_kernel`` (proj/src/scheme.cpp:59-105), ``kinetic_convolve``
(proj/src/scheme.cpp:107-146), ``step_fully_discrete`` (:148-164),
``evolve`` (:208-272) and ``split_step_nd`` (proj/src/splitting.cpp:37-99).
Lines are numpy arrays (host) or torch CUDA tensors (device-resident);
every compute call runs on the B200 through ``lib/liblaxol_b200.so``.
Errors raise the mirrors of the reference's exceptions (InvalidInput,
EvaluationError).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import (DIRECT_PLAIN, DIRECT_SCREENED, ENGINE_DIRECT, ENGINE_FAST, ENGINE_RELAXED, FAST_CHAINED, FAST_STATS_CHECK, FAST_STATS_VALID, EvaluationError,  # noqa: F401
                    InvalidInput, check)


def _ptr(x) -> int | None:
    """Raw data pointer of a numpy array or torch tensor (None passes NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise InvalidInput("array must be C-contiguous")
        return x.ctypes.data
    if not x.is_contiguous():
        raise InvalidInput("tensor must be contiguous")
    return x.data_ptr()


def _stream_ptr(stream) -> int | None:
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


@dataclass
class Kernel:
    """Sampled kinetic cost (proj/include/laxol/scheme.hpp:34-42): window of
    2n+1 samples at grid displacements first..first+2n."""

    window: np.ndarray
    first: int
    argmin_index: int
    center_index: int
    n_space: int
    tau: float
    drift: float
    delta: float = 0.0  # fast-path slope-estimate tolerance (displacement units)


@dataclass
class SchemeParams:
    """proj/include/laxol/scheme.hpp:17-26"""

    n_space: int
    tau: float
    eta: float = 0.0
    h0: float = 1.0
    arrival: bool = True  # PotentialSampling::Arrival (V at t + tau)

    @property
    def epsilon(self) -> float:
        return 1.0 / float(self.n_space)


def validate(params: SchemeParams) -> None:
    """proj/src/scheme.cpp:39-53 (AntiCflMode::Fail)."""
    if params.n_space < 1:
        raise InvalidInput("SchemeParams: n_space must be >= 1")
    if not params.tau > 0.0:
        raise InvalidInput("SchemeParams: tau must be positive")
    if params.eta < 0.0:
        raise InvalidInput("SchemeParams: eta must be >= 0")
    if not params.h0 > 0.0:
        raise InvalidInput("SchemeParams: h0 must be positive")
    if params.epsilon / params.tau >= params.h0:
        raise InvalidInput("SchemeParams: epsilon/tau violates the bound epsilon/tau < h0")


class Device:
    """One laxol_b200 context (lob_ctx) on one CUDA device."""

    def __init__(self, device: int = 0):
        self.lib = _capi.load()
        h = ctypes.c_void_p()
        st = self.lib.lob_ctx_create(int(device), ctypes.byref(h))
        if st != 0:
            raise _capi.CudaError(f"lob_ctx_create(device={device}) failed with status {st} "
                                  "(no CUDA device? there is no CPU fallback)")
        self.ctx = h
        self.device = device

    def close(self):
        if self.ctx:
            self.lib.lob_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, where):
        check(st, self.ctx, where)

    @property
    def launches(self) -> int:
        return int(self.lib.lob_launch_count(self.ctx))

    def set_evolve_resident(self, on: bool) -> None:
        """evolve through the on-chip resident kernels (K2R / K2C) where the lines fit (default)."""
        self._check(self.lib.lob_ctx_set_evolve_resident(self.ctx, int(bool(on))), "lob_ctx_set_evolve_resident")

    def set_fast_line(self, on: bool) -> None:
        """Short lines (n <= 2048) on the whole-line fast kernel (K2L, default) or the tiled one."""
        self._check(self.lib.lob_ctx_set_fast_line(self.ctx, int(on)), "lob_ctx_set_fast_line")

    def set_direct_mode(self, mode: int) -> None:
        """DIRECT_SCREENED (default: fp32 screen + fp64 re-evaluation) or DIRECT_PLAIN."""
        self._check(self.lib.lob_ctx_set_direct_mode(self.ctx, int(mode)), "lob_ctx_set_direct_mode")

    def direct_stats(self, reset: bool = True) -> dict:
        """Screened-K1 counters since the last reset: outputs swept in full fp64
        and fp64 candidates re-evaluated."""
        f, c = ctypes.c_uint64(), ctypes.c_uint64()
        self._check(self.lib.lob_direct_stats(self.ctx, ctypes.byref(f), ctypes.byref(c), int(reset)),
                    "lob_direct_stats")
        return {"full_outputs": int(f.value), "fp64_candidates": int(c.value)}

    def direct_fallbacks(self, reset: bool = True) -> int:
        """Outputs the screened K1 swept in full fp64 since the last reset."""
        return self.direct_stats(reset)["full_outputs"]

    # ---- kernels -----------------------------------------------------------
    def build_kernel(self, n_space: int, tau: float, drift: float) -> Kernel:
        """Host build_kernel for mechanical(drift) (proj/src/scheme.cpp:59-105)."""
        validate(SchemeParams(n_space, tau))
        win = np.empty(2 * n_space + 1, dtype=np.float64)
        first = ctypes.c_int64()
        arg = ctypes.c_int64()
        delta = ctypes.c_double()
        st = self.lib.lob_kernel_mech_host(self.ctx, n_space, tau, drift, win.ctypes.data,
                                           ctypes.byref(first), ctypes.byref(arg), ctypes.byref(delta))
        self._check(st, "build_kernel")
        return Kernel(win, int(first.value), int(arg.value), int(first.value) + n_space, n_space,
                      tau, drift, float(delta.value))

    @staticmethod
    def build_kernel_tabulated(n_space: int, tau: float, samples, v0: float, dv: float) -> Kernel:
        """Host build_kernel for tabulated(samples, v0, dv) (proj/src/scheme.cpp:59-105)."""
        smp = np.ascontiguousarray(samples, np.float64)
        win = np.empty(2 * n_space + 1, dtype=np.float64)
        first, arg = ctypes.c_int64(), ctypes.c_int64()
        st = _capi.load().lob_kernel_tabulated_host(None, n_space, tau, smp.ctypes.data, smp.size, v0, dv,
                                                     win.ctypes.data, ctypes.byref(first), ctypes.byref(arg))
        check(st, None, "build_kernel_tabulated")
        return Kernel(win, int(first.value), int(arg.value), int(first.value) + n_space, n_space, tau, float("nan"))

    def direct_f64(self, u, out, ktab, first, tv=None, ktab_stride=0, tv_stride=0, stream=None):
        lines, n = u.shape
        st = self.lib.lob_minplus_direct_f64(self.ctx, _ptr(u), _ptr(out), lines, n, _ptr(ktab),
                                             ktab_stride, _ptr(first), _ptr(tv), tv_stride,
                                             _stream_ptr(stream))
        self._check(st, "lob_minplus_direct_f64")

    def direct_f32(self, u, out, ktab, first, ktab_stride=0, stream=None):
        lines, n = u.shape
        st = self.lib.lob_minplus_direct_f32(self.ctx, _ptr(u), _ptr(out), lines, n, _ptr(ktab),
                                             ktab_stride, _ptr(first), _stream_ptr(stream))
        self._check(st, "lob_minplus_direct_f32")

    def window_f64(self, u, out, n_space, ktab, first, tv=None, ktab_stride=0, tv_stride=0,
                   stream=None):
        lines, m = u.shape
        st = self.lib.lob_minplus_window_f64(self.ctx, _ptr(u), _ptr(out), lines, m, n_space,
                                             _ptr(ktab), ktab_stride, _ptr(first), _ptr(tv),
                                             tv_stride, _stream_ptr(stream))
        self._check(st, "lob_minplus_window_f64")

    def fast_workspace_bytes(self, lines: int, n: int) -> int:
        b = ctypes.c_size_t()
        st = self.lib.lob_fast_workspace_bytes(lines, n, ctypes.byref(b))
        self._check(st, "lob_fast_workspace_bytes")
        return int(b.value)

    def fast_f64(self, u, out, drift, tau, tv=None, tv_stride=0, eta=0.0, blocks=None,
                 workspace=None, flags=0, stream=None):
        lines, n = u.shape
        ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
        st = self.lib.lob_minplus_fast_f64(self.ctx, _ptr(u), _ptr(out), lines, n, _ptr(drift),
                                           float(tau), _ptr(tv), tv_stride, float(eta), _ptr(blocks),
                                           _ptr(workspace), ws_bytes, int(flags), _stream_ptr(stream))
        self._check(st, "lob_minplus_fast_f64")

    def fast_window_f64(self, u, out, ktab, first, tau, tv=None, tv_stride=0, eta=0.0, blocks=None,
                        workspace=None, flags=0, ktab_stride=0, stream=None):
        """K2 over any convex kernel window (lob_minplus_fast_window_f64): the engine for
        kinetic_convolve's Kernel (mechanical or tabulated)."""
        lines, n = u.shape
        ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
        st = self.lib.lob_minplus_fast_window_f64(self.ctx, _ptr(u), _ptr(out), lines, n, _ptr(ktab), ktab_stride,
                                                  _ptr(first), float(tau), _ptr(tv), tv_stride, float(eta),
                                                  _ptr(blocks), _ptr(workspace), ws_bytes, int(flags),
                                                  _stream_ptr(stream))
        self._check(st, "lob_minplus_fast_window_f64")

    def set_fast_delta(self, delta: float = float("nan")) -> None:
        """Diagnostic: override the fast engine's rounding tolerance delta (NaN: the computed bound)."""
        self._check(self.lib.lob_ctx_set_fast_delta(self.ctx, float(delta)), "lob_ctx_set_fast_delta")

    FAST_COUNTER_KEYS = ["missed_outputs", "sources", "queued_candidates", "queued_intervals", "tiles", "tiles_k_unstaged",
                         "k_range_sum", "direct_tiles_gate", "direct_tiles_heavy", "chain_timeouts",
                         "stats_check_mismatches", "stale_line_constants"]

    def fast_counters(self, workspace, lines: int, n: int) -> dict:
        """The fast engine's work counters (include/laxol_b200.h, lob_fast_diagnostics)."""
        v = (ctypes.c_uint64 * 16)()
        st = self.lib.lob_fast_diagnostics(self.ctx, _ptr(workspace), lines, n, v)
        self._check(st, "lob_fast_diagnostics")
        return {k: int(v[i]) for i, k in enumerate(self.FAST_COUNTER_KEYS)}

    def fast_diagnostics(self, workspace, lines: int, n: int) -> int:
        return self.fast_counters(workspace, lines, n)["missed_outputs"]

    def split_step_2d(self, u, out, tmp, tau, drift1, drift2, a1=None, a2=None, b=0.0,
                      engine=ENGINE_DIRECT, workspace=None, stream=None):
        n = u.shape[0]
        ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
        st = self.lib.lob_split_step_2d_f64(self.ctx, _ptr(u), _ptr(out), _ptr(tmp), n, float(tau),
                                            float(drift1), float(drift2), _ptr(a1), _ptr(a2),
                                            float(b), int(engine), _ptr(workspace), ws_bytes,
                                            _stream_ptr(stream))
        self._check(st, "lob_split_step_2d_f64")

    def split_step_nd(self, u, out, tmp, rank, n, tau, kernels=None, drifts=None, tv=None, eta=0.0,
                      engine=ENGINE_DIRECT, workspace=None, stream=None):
        """split_step_nd (proj/src/splitting.cpp:37-99) of a periodic rank-`rank` tensor (n^rank
        device doubles).  kernels: per-axis Kernel windows (direct / relaxed engines); drifts:
        per-axis mechanical drifts (fast engine); tv: device tau*V of every point or None."""
        import torch
        kt = fr = dr = None
        if kernels is not None:
            kt = torch.from_numpy(np.concatenate([k.window for k in kernels])).to(u.device)
            fr = (ctypes.c_int64 * rank)(*[int(k.first) for k in kernels])
        if drifts is not None:
            dr = (ctypes.c_double * rank)(*[float(d) for d in drifts])
        ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
        st = self.lib.lob_split_step_nd_f64(self.ctx, _ptr(u), _ptr(out), _ptr(tmp), int(rank), int(n), float(tau),
                                            _ptr(kt), fr, dr, _ptr(tv), float(eta), int(engine), _ptr(workspace),
                                            ws_bytes, _stream_ptr(stream))
        self._check(st, "lob_split_step_nd_f64")

    def split_step_nd_window(self, u, out, tmp, dims, n, tau, kernels, tv=None, stream=None):
        """split_step_nd of a windowed tensor (walls) of shape dims (device doubles, row-major)."""
        import torch
        rank = len(dims)
        kt = torch.from_numpy(np.concatenate([k.window for k in kernels])).to(u.device)
        fr = (ctypes.c_int64 * rank)(*[int(k.first) for k in kernels])
        dm = (ctypes.c_int64 * rank)(*[int(x) for x in dims])
        st = self.lib.lob_split_step_nd_window_f64(self.ctx, _ptr(u), _ptr(out), _ptr(tmp), rank, dm, int(n),
                                                   float(tau), _ptr(kt), fr, _ptr(tv), _stream_ptr(stream))
        self._check(st, "lob_split_step_nd_window_f64")

    def evolve(self, u, scratch, drift, tau, steps, tv=None, tv_stride=0, eta=0.0,
               engine=ENGINE_FAST, step_drift=None, step_blocks=None, workspace=None, stream=None):
        lines, n = u.shape
        done = ctypes.c_int64()
        ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
        st = self.lib.lob_evolve_f64(self.ctx, _ptr(u), _ptr(scratch), lines, n, _ptr(drift),
                                     float(tau), _ptr(tv), tv_stride, float(eta), int(engine),
                                     int(steps), _ptr(step_drift), _ptr(step_blocks),
                                     ctypes.byref(done), _ptr(workspace), ws_bytes,
                                     _stream_ptr(stream))
        self._check(st, "lob_evolve_f64")
        return int(done.value)

    def step_host(self, u: np.ndarray, drift: np.ndarray, tau: float, tv=None, tv_stride=0,
                  eta=0.0, engine=ENGINE_FAST, out=None, blocks=None) -> np.ndarray:
        lines, n = u.shape
        if out is None:
            out = np.empty_like(u)
        st = self.lib.lob_step_host_f64(self.ctx, _ptr(u), _ptr(out), lines, n, _ptr(drift),
                                        float(tau), _ptr(tv), tv_stride, float(eta), int(engine),
                                        _ptr(blocks))
        self._check(st, "lob_step_host_f64")
        return out

    def block_counts(self, u, blocks, eta=0.0, stream=None):
        lines, n = u.shape
        st = self.lib.lob_block_counts(self.ctx, _ptr(u), lines, n, float(eta), _ptr(blocks),
                                       _stream_ptr(stream))
        self._check(st, "lob_block_counts")

    # ---- the reference's relaxed fast engine, eta > 0 (proj/src/minplus.cpp:152-276) ----
    def relaxed_workspace_bytes(self, lines: int, n: int) -> int:
        b = ctypes.c_size_t()
        self._check(self.lib.lob_relaxed_workspace_bytes(lines, n, ctypes.byref(b)), "lob_relaxed_workspace_bytes")
        return int(b.value)

    def relaxed_f64(self, u, out, ktab, first, eta, tv=None, ktab_stride=0, tv_stride=0, blocks=None,
                    workspace=None, stream=None):
        lines, n = u.shape
        if workspace is None:
            import torch
            workspace = torch.empty(self.relaxed_workspace_bytes(lines, n), dtype=torch.uint8, device=u.device)
        ws_bytes = workspace.numel() * workspace.element_size()
        st = self.lib.lob_minplus_relaxed_f64(self.ctx, _ptr(u), _ptr(out), lines, n, _ptr(ktab), ktab_stride,
                                              _ptr(first), _ptr(tv), tv_stride, float(eta), _ptr(blocks),
                                              _ptr(workspace), ws_bytes, _stream_ptr(stream))
        self._check(st, "lob_minplus_relaxed_f64")

    # ---- min-plus primitives on plain sequences (proj/include/laxol/minplus.hpp) ----
    def conv_naive(self, f, g, out, stream=None):
        st = self.lib.lob_minplus_conv_naive_f64(self.ctx, _ptr(f), f.numel(), _ptr(g), g.numel(), _ptr(out),
                                                 _stream_ptr(stream))
        self._check(st, "lob_minplus_conv_naive_f64")

    def decompose(self, u, eta=0.0, stream=None):
        """[(kind, start, end)] with kind 0 convex / 1 concave (proj/src/minplus.cpp:152-188)."""
        m = u.numel()
        cap = max(m, 1)
        kinds = np.empty(cap, np.int32)
        starts = np.empty(cap, np.int64)
        ends = np.empty(cap, np.int64)
        cnt = ctypes.c_int64()
        st = self.lib.lob_decompose_f64(self.ctx, _ptr(u), m, float(eta), kinds.ctypes.data, starts.ctypes.data,
                                        ends.ctypes.data, cap, ctypes.byref(cnt), _stream_ptr(stream))
        self._check(st, "lob_decompose_f64")
        c = int(cnt.value)
        return kinds[:c], starts[:c], ends[:c]

    def conv_fast(self, kern, u, out, eta=0.0, stream=None) -> int:
        """conv_fast (proj/src/minplus.cpp:190-252); returns the block count."""
        b = ctypes.c_int64()
        st = self.lib.lob_conv_fast_f64(self.ctx, _ptr(kern), kern.numel(), _ptr(u), u.numel(), float(eta),
                                        _ptr(out), ctypes.byref(b), _stream_ptr(stream))
        self._check(st, "lob_conv_fast_f64")
        return int(b.value)

    # ---- step_semidiscrete (proj/src/scheme.cpp:166-206) -----------------------
    def step_semidiscrete(self, u, out, ktab, first, t, tau, potential=None, quad_points=1, periodic=True,
                          origin=0.0, n_space=None, stream=None):
        """One semi-discrete step of lines x m device samples (periodic: m == n_space)."""
        lines, m = u.shape
        n = m if n_space is None else int(n_space)
        pot = potential_zero() if potential is None else potential
        p = _capi.LobPotential(pot["kind"], pot["value"], pot["offset"], pot["amplitude"], pot["frequency"],
                               pot["tmod"], pot["omega"])
        st = self.lib.lob_step_semidiscrete_f64(self.ctx, _ptr(u), _ptr(out), lines, m, n, int(periodic),
                                                float(origin), _ptr(ktab), int(first), float(t), float(tau),
                                                ctypes.byref(p), int(quad_points), _stream_ptr(stream))
        self._check(st, "lob_step_semidiscrete_f64")

    # ---- weak-KAM consumers (proj/src/weakkam.cpp; include/laxol_b200.h) ----
    def minplus_gemm(self, a, b, out, stream=None):
        """out = a (x) b in the min-plus semiring (minplus_product / minplus_apply)."""
        m, k = a.shape
        k2, n = b.shape
        if k2 != k or tuple(out.shape) != (m, n):
            raise InvalidInput("minplus_gemm: shape mismatch")
        st = self.lib.lob_minplus_gemm_f64(self.ctx, _ptr(a), a.stride(0), _ptr(b), b.stride(0), _ptr(out),
                                           out.stride(0), m, n, k, _stream_ptr(stream))
        self._check(st, "lob_minplus_gemm_f64")

    @staticmethod
    def period_kinetic(kernel: "Kernel") -> np.ndarray:
        """kin[r] = min over displacements = r (mod n) in the window (proj/src/weakkam.cpp:106-118)."""
        w = np.ascontiguousarray(kernel.window, np.float64)
        n = (w.size - 1) // 2
        kinc = np.empty(n)
        st = _capi.load().lob_period_kinetic_host(w.ctypes.data, int(kernel.first), n, kinc.ctypes.data)
        _capi.check(st, None, "lob_period_kinetic_host")
        return kinc

    def period_matrix(self, kinc, tvs, ell, out, scratch, stream=None):
        """build_period_matrix (proj/src/weakkam.cpp:88-128) on device buffers."""
        n = kinc.shape[0]
        st = self.lib.lob_period_matrix_f64(self.ctx, _ptr(kinc), _ptr(tvs), n, int(ell), _ptr(out),
                                            _ptr(scratch), _stream_ptr(stream))
        self._check(st, "lob_period_matrix_f64")

    def eigenvalue_karp(self, m, stream=None) -> float:
        lam = ctypes.c_double()
        st = self.lib.lob_eigenvalue_karp_f64(self.ctx, _ptr(m), m.shape[0], ctypes.byref(lam), _stream_ptr(stream))
        self._check(st, "lob_eigenvalue_karp_f64")
        return lam.value

    @staticmethod
    def _tvs(tvs):
        if tvs is None:
            return None, 0
        t = np.ascontiguousarray(np.atleast_2d(tvs), np.float64)
        return t, t.shape[0]

    def hbar_drift_host(self, u0, drift, tau, tvs=None, engine=ENGINE_FAST, max_periods=100, tol=1e-10):
        """estimate_hbar_drift (proj/src/weakkam.cpp:43-86) of one periodic line (host arrays);
        tvs: None, one table, or one rounded tau*V table per in-period step."""
        u0 = np.ascontiguousarray(u0, np.float64)
        t, nt = self._tvs(tvs)
        hb, res, ns, cv = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64(), ctypes.c_int()
        uf = np.empty_like(u0)
        st = self.lib.lob_hbar_drift_host_f64(self.ctx, u0.ctypes.data, u0.size, float(drift), float(tau),
                                              None if t is None else t.ctypes.data, nt, int(engine),
                                              int(max_periods), float(tol), ctypes.byref(hb),
                                              ctypes.byref(res), ctypes.byref(ns), ctypes.byref(cv),
                                              uf.ctypes.data)
        self._check(st, "lob_hbar_drift_host_f64")
        return {"h_bar": hb.value, "residual": res.value, "n_steps": ns.value, "converged": bool(cv.value),
                "u": uf}

    def fixed_point_residual_host(self, u, drift, tau, h_bar, tvs=None, engine=ENGINE_FAST) -> float:
        u = np.ascontiguousarray(u, np.float64)
        t, nt = self._tvs(tvs)
        r = ctypes.c_double()
        st = self.lib.lob_fixed_point_residual_host_f64(self.ctx, u.ctypes.data, u.size, float(h_bar),
                                                        float(drift), float(tau),
                                                        None if t is None else t.ctypes.data, nt, int(engine),
                                                        ctypes.byref(r))
        self._check(st, "lob_fixed_point_residual_host_f64")
        return r.value

    def bench_fp64(self):
        a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        st = self.lib.lob_bench_fp64(self.ctx, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
        self._check(st, "lob_bench_fp64")
        return {"minplus_cand_per_s": a.value, "dadd_ops_per_s": b.value, "sm_clock_ghz": c.value}


# ---- built-in potentials (proj/src/hamiltonian.cpp:77-117) --------------------
def potential_zero() -> dict:
    return dict(kind=_capi.POTENTIAL_ZERO, value=0.0, offset=0.0, amplitude=0.0, frequency=1,
                tmod=_capi.TMOD_NONE, omega=0.0)


def potential_const(c: float) -> dict:
    return dict(potential_zero(), kind=_capi.POTENTIAL_CONST, value=float(c))


def potential_cosine(offset: float, amplitude: float, frequency: int, tmod: int = 0, omega: float = 0.0) -> dict:
    if frequency < 1:
        raise InvalidInput("potential_cosine: frequency must be >= 1")
    return dict(potential_zero(), kind=_capi.POTENTIAL_COSINE, offset=float(offset), amplitude=float(amplitude),
                frequency=int(frequency), tmod=int(tmod), omega=float(omega))


# ---- synthetic workloads (include/laxol_b200_configs.h) ---------------------

def gen_sin(n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    _capi.load_configs().lob_gen_sin(n, out.ctypes.data)
    return out


def gen_cos(n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    _capi.load_configs().lob_gen_cos(n, out.ctypes.data)
    return out


def gen_potential(kind: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    _capi.load_configs().lob_gen_potential(int(kind), n, out.ctypes.data)
    return out


def gen_c2_drifts(lines: int = 256) -> np.ndarray:
    out = np.empty(lines, np.float64)
    _capi.load_configs().lob_gen_c2_drifts(lines, out.ctypes.data)
    return out


def gen_c3_lines(line0: int, lines: int, n: int = 4096, seed0: int = 1000) -> np.ndarray:
    out = np.empty((lines, n), np.float64)
    _capi.load_configs().lob_gen_c3_lines(line0, lines, n, seed0, out.ctypes.data)
    return out


def gen_c4_u0(n: int = 2048) -> np.ndarray:
    out = np.empty((n, n), np.float64)
    _capi.load_configs().lob_gen_c4_u0(n, out.ctypes.data)
    return out


def c4_time_term(t: float) -> float:
    return float(_capi.load_configs().lob_c4_time_term(float(t)))


def gen_c5_lines(line0: int, lines: int, n: int = 1 << 20, seed0: int = 5000,
                 nthreads: int = 0) -> np.ndarray:
    import os

    out = np.empty((lines, n), np.float64)
    nt = nthreads or (os.cpu_count() or 1)
    _capi.load_configs().lob_gen_c5_lines(line0, lines, n, seed0, out.ctypes.data, nt)
    return out


def tau_v(v: np.ndarray, tau: float) -> np.ndarray:
    """tau*V rounded once (the product in proj/src/scheme.cpp:161)."""
    return np.multiply(float(tau), v)


def llround(x: float) -> int:
    """C llround: half away from zero."""
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))
