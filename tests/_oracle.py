"""Test-only loaders for the CPU checkers under oracle/ (never the product).

oracle():    the plain-C restatement, oracle/_build/liblaxol_oracle.so
reference(): the unmodified reference library built from /root/reference
             sources + our extern "C" shim, oracle/_ref/liblaxol_ref.so
"""
import ctypes
import os
import subprocess
from ctypes import POINTER, c_char_p, c_double, c_int, c_int64, c_void_p

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liblaxol_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "liblaxol_ref.so")

_P = c_void_p


def _build_oracle():
    subprocess.run(["make", "-s", "-f", os.path.join(ROOT, "oracle", "Makefile"), "oracle"],
                   check=True, cwd=ROOT)


class Oracle:
    def __init__(self, lib):
        self.lib = lib
        sig = {
            "orc_kernel_mech": (c_int, [c_int, c_double, c_double, _P, POINTER(c_int64), POINTER(c_int64)]),
            "orc_direct_f64": (None, [_P, _P, c_int64, c_int64, _P, c_int64, _P, _P, c_int64, c_int]),
            "orc_direct_f32": (None, [_P, _P, c_int64, c_int64, _P, c_int64, _P, c_int]),
            "orc_window_f64": (c_int, [_P, c_int64, c_int64, _P, c_int64, _P]),
            "orc_conv_naive": (None, [_P, c_int64, _P, c_int64, _P]),
            "orc_decompose_count": (c_int64, [_P, c_int64, c_double, c_int]),
            "orc_line_blocks": (c_int64, [_P, c_int64, c_double, c_int]),
            "orc_split2d_f64": (None, [_P, _P, c_int64, c_int64, _P, c_int64, _P, c_int64, _P, c_int]),
            "orc_drift": (c_double, [_P, _P, c_int64, POINTER(c_int)]),
            "orc_tau_v": (None, [_P, c_double, c_int64, _P]),
        }
        for k, (r, a) in sig.items():
            f = getattr(lib, k)
            f.restype, f.argtypes = r, a

    def kernel(self, n, tau, drift):
        w = np.empty(2 * n + 1)
        first, arg = c_int64(), c_int64()
        st = self.lib.orc_kernel_mech(n, tau, drift, w.ctypes.data, ctypes.byref(first), ctypes.byref(arg))
        return w, first.value, arg.value, st

    def direct(self, u, ktab, first, tv=None, ktab_stride=0, tv_stride=0, nthreads=0):
        u = np.ascontiguousarray(u, np.float64)
        lines, n = u.shape
        out = np.empty_like(u)
        first = np.ascontiguousarray(np.broadcast_to(np.asarray(first, np.int64), (lines,)))
        self.lib.orc_direct_f64(u.ctypes.data, out.ctypes.data, lines, n, ktab.ctypes.data, ktab_stride,
                                first.ctypes.data, None if tv is None else tv.ctypes.data, tv_stride,
                                nthreads)
        return out

    def direct_f32(self, u, ktab, first, ktab_stride=0, nthreads=0):
        u = np.ascontiguousarray(u, np.float32)
        lines, n = u.shape
        out = np.empty_like(u)
        first = np.ascontiguousarray(np.broadcast_to(np.asarray(first, np.int64), (lines,)))
        self.lib.orc_direct_f32(u.ctypes.data, out.ctypes.data, lines, n, ktab.ctypes.data, ktab_stride,
                                first.ctypes.data, nthreads)
        return out

    def window(self, u, n, ktab, first):
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty_like(u)
        st = self.lib.orc_window_f64(u.ctypes.data, u.size, n, ktab.ctypes.data, first, out.ctypes.data)
        return out, st

    def conv_naive(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.empty(a.size + b.size - 1)
        self.lib.orc_conv_naive(a.ctypes.data, a.size, b.ctypes.data, b.size, out.ctypes.data)
        return out

    def decompose_count(self, v, eta=0.0, capped=False):
        v = np.ascontiguousarray(v, np.float64)
        return int(self.lib.orc_decompose_count(v.ctypes.data, v.size, eta, int(capped)))

    def line_blocks(self, u, eta=0.0, capped=False):
        u = np.ascontiguousarray(u, np.float64)
        return int(self.lib.orc_line_blocks(u.ctypes.data, u.size, eta, int(capped)))

    def split2d(self, u, k1, first1, k2, first2, tv=None, nthreads=0):
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty_like(u)
        n1, n2 = u.shape
        self.lib.orc_split2d_f64(u.ctypes.data, out.ctypes.data, n1, n2, k1.ctypes.data, first1,
                                 k2.ctypes.data, first2, None if tv is None else tv.ctypes.data, nthreads)
        return out

    def drift(self, nxt, u):
        fin = c_int()
        d = self.lib.orc_drift(np.ascontiguousarray(nxt).ctypes.data, np.ascontiguousarray(u).ctypes.data,
                               u.size, ctypes.byref(fin))
        return d, bool(fin.value)


class Reference:
    """The reference library itself (oracle/_ref), via oracle/ref_shim.cpp."""

    def __init__(self, lib):
        self.lib = lib
        sig = {
            "ref_last_error": (c_char_p, []),
            "ref_set_max_threads": (None, [c_int]),
            "ref_kernel_mech": (c_int, [c_int, c_double, c_double, _P, POINTER(c_int64), POINTER(c_int64)]),
            "ref_kinetic_convolve": (c_int, [_P, c_int64, c_int, c_int, c_double, c_double, c_double, c_int, _P,
                                             POINTER(c_int64)]),
            "ref_step_lines": (c_int, [_P, c_int64, c_int, c_double, _P, _P, c_double, c_double, c_int, c_int,
                                       _P, _P]),
            "ref_evolve": (c_int, [_P, c_int, c_double, c_double, _P, c_double, c_int64, c_double, c_int, _P, _P,
                                   _P, POINTER(c_int)]),
            "ref_split_step_2d": (c_int, [_P, c_int64, c_int64, c_int, c_double, c_double, c_double, c_int,
                                          c_double, c_int, _P]),
            "ref_decompose": (c_int64, [_P, c_int64, c_double, _P, _P, _P, c_int64]),
            "ref_conv": (c_int, [c_int, _P, c_int64, _P, c_int64, c_double, _P, _P]),
            "ref_minplus_product": (c_int, [_P, _P, c_int64, _P]),
            "ref_split_step_nd": (c_int, [_P, c_int, c_int, c_double, _P, _P, c_double, c_double, _P]),
            "ref_split_step_nd_window": (c_int, [_P, c_int, _P, _P, c_int, c_double, _P, _P, c_double, _P]),
            "ref_kernel_tabulated": (c_int, [c_int, c_double, _P, c_int64, c_double, c_double, _P, POINTER(c_int64),
                                             POINTER(c_int64)]),
            "ref_convolve_tabulated": (c_int, [_P, c_int, c_double, _P, c_int64, c_double, c_double, c_double, c_int,
                                               _P, POINTER(c_int64)]),
            "ref_step_semidiscrete": (c_int, [_P, c_int64, c_int, c_double, c_int, c_double, c_double, c_int,
                                              c_double, c_double, c_double, c_int, c_int, c_double, c_double,
                                              c_int, _P]),
            "ref_minplus_apply": (c_int, [_P, c_int64, _P, _P]),
            "ref_eigenvalue_karp": (c_int, [_P, c_int64, POINTER(c_double)]),
            "ref_build_period_matrix": (c_int, [c_int, c_double, c_double, _P, c_int64, _P]),
            "ref_estimate_hbar_drift": (c_int, [_P, c_int, c_double, c_double, _P, c_int64, c_int, c_double,
                                                POINTER(c_double), POINTER(c_double), POINTER(c_int64),
                                                POINTER(c_int)]),
            "ref_fixed_point_residual": (c_int, [_P, c_int, c_double, c_double, _P, c_int64, c_double,
                                                 POINTER(c_double)]),
        }
        for k, (r, a) in sig.items():
            f = getattr(lib, k)
            f.restype, f.argtypes = r, a

    def err(self):
        return self.lib.ref_last_error().decode()

    # the synthetic-workload generators compiled into the reference shim (oracle/Makefile), so
    # a reference-only process (bench.py --impl reference) maps no product library
    def gen_c2_drifts(self, lines=256):
        out = np.empty(lines, np.float64)
        self.lib.lob_gen_c2_drifts(ctypes.c_int64(lines), out.ctypes.data_as(ctypes.c_void_p))
        return out

    def gen_potential(self, kind, n):
        out = np.empty(n, np.float64)
        self.lib.lob_gen_potential(ctypes.c_int(kind), ctypes.c_int64(n), out.ctypes.data_as(ctypes.c_void_p))
        return out

    def kernel(self, n, tau, drift):
        w = np.empty(2 * n + 1)
        c, a = c_int64(), c_int64()
        st = self.lib.ref_kernel_mech(n, tau, drift, w.ctypes.data, ctypes.byref(c), ctypes.byref(a))
        return w, c.value - n, a.value, st

    def kinetic_convolve(self, u, n_space, tau, drift, eta=0.0, engine=0, periodic=True):
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty(n_space if periodic else u.size)
        blocks = c_int64()
        st = self.lib.ref_kinetic_convolve(u.ctypes.data, u.size, int(periodic), n_space, tau, drift, eta,
                                           engine, out.ctypes.data, ctypes.byref(blocks))
        return out, blocks.value, st

    def step_lines(self, u, tau, drifts, v=None, t=0.0, eta=0.0, engine=0, nthreads=1, want_blocks=True):
        u = np.ascontiguousarray(u, np.float64)
        lines, n = u.shape
        drifts = np.ascontiguousarray(np.broadcast_to(np.asarray(drifts, np.float64), (lines,)))
        out = np.empty_like(u)
        blocks = np.empty(lines, np.int64)
        st = self.lib.ref_step_lines(u.ctypes.data, lines, n, tau, drifts.ctypes.data,
                                     None if v is None else np.ascontiguousarray(v).ctypes.data, t, eta, engine,
                                     nthreads, out.ctypes.data, blocks.ctypes.data if want_blocks else None)
        if st:
            raise RuntimeError(self.err())
        return out, blocks

    def evolve(self, u0, tau, drift, v, steps, t0=0.0, eta=0.0, engine=0):
        u0 = np.ascontiguousarray(u0, np.float64)
        n = u0.size
        uf = np.empty(n)
        dr = np.empty(max(steps, 1))
        bl = np.empty(max(steps, 1), np.int64)
        comp = c_int()
        st = self.lib.ref_evolve(u0.ctypes.data, n, tau, drift, None if v is None else v.ctypes.data, t0, steps,
                                 eta, engine, uf.ctypes.data, dr.ctypes.data, bl.ctypes.data, ctypes.byref(comp))
        if st:
            raise RuntimeError(self.err())
        return uf, dr[:steps], bl[:steps], bool(comp.value)

    def split_step_2d(self, u, tau, d1, d2, pot_kind=0, t=0.0, periodic=True):
        u = np.ascontiguousarray(u, np.float64)
        n1, n2 = u.shape
        out = np.empty_like(u)
        st = self.lib.ref_split_step_2d(u.ctypes.data, n1, n2, n1, tau, d1, d2, pot_kind, t, int(periodic),
                                        out.ctypes.data)
        if st:
            raise RuntimeError(self.err())
        return out

    def decompose(self, v, eta=0.0):
        v = np.ascontiguousarray(v, np.float64)
        cap = v.size + 1
        kinds = np.empty(cap, np.int32)
        starts = np.empty(cap, np.int64)
        ends = np.empty(cap, np.int64)
        c = self.lib.ref_decompose(v.ctypes.data, v.size, eta, kinds.ctypes.data, starts.ctypes.data,
                                   ends.ctypes.data, cap)
        return int(c), kinds[:c], starts[:c], ends[:c]

    def conv(self, which, a, b, eta=0.0):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.empty(a.size + b.size - 1)
        blocks = c_int64()
        st = self.lib.ref_conv(which, a.ctypes.data, a.size, b.ctypes.data, b.size, eta, out.ctypes.data,
                               ctypes.byref(blocks))
        return out, blocks.value, st

    def split_step_nd(self, u, rank, n, tau, drifts, vtab=None, t=0.0, eta=0.0):
        u = np.ascontiguousarray(u, np.float64).ravel()
        d = np.ascontiguousarray(drifts, np.float64)
        out = np.empty_like(u)
        st = self.lib.ref_split_step_nd(u.ctypes.data, rank, n, tau, d.ctypes.data,
                                        None if vtab is None else np.ascontiguousarray(vtab).ctypes.data, t, eta,
                                        out.ctypes.data)
        if st:
            raise RuntimeError(self.err())
        return out

    def split_step_nd_window(self, u, n_space, tau, drifts, origins, vtab=None, t=0.0):
        u = np.ascontiguousarray(u, np.float64)
        dims = np.ascontiguousarray(u.shape, np.int64)
        org = np.ascontiguousarray(origins, np.float64)
        d = np.ascontiguousarray(drifts, np.float64)
        out = np.empty(u.size)
        st = self.lib.ref_split_step_nd_window(u.ctypes.data, u.ndim, dims.ctypes.data, org.ctypes.data, n_space,
                                               tau, d.ctypes.data,
                                               None if vtab is None else np.ascontiguousarray(vtab).ctypes.data,
                                               t, out.ctypes.data)
        return out, st

    def kernel_tabulated(self, n, tau, samples, v0, dv):
        smp = np.ascontiguousarray(samples, np.float64)
        w = np.empty(2 * n + 1)
        c, a = c_int64(), c_int64()
        st = self.lib.ref_kernel_tabulated(n, tau, smp.ctypes.data, smp.size, v0, dv, w.ctypes.data,
                                           ctypes.byref(c), ctypes.byref(a))
        return w, c.value - n, a.value, st

    def convolve_tabulated(self, u, tau, samples, v0, dv, eta=0.0, engine=0):
        u = np.ascontiguousarray(u, np.float64)
        smp = np.ascontiguousarray(samples, np.float64)
        out = np.empty_like(u)
        b = c_int64()
        st = self.lib.ref_convolve_tabulated(u.ctypes.data, u.size, tau, smp.ctypes.data, smp.size, v0, dv, eta,
                                             engine, out.ctypes.data, ctypes.byref(b))
        return out, b.value, st

    def step_semidiscrete(self, u, n_space, tau, drift, pot, t, q, periodic=True, origin=0.0):
        """pot: dict(kind, value, offset, amplitude, frequency, tmod, omega) (api.potential_*)."""
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty(n_space if periodic else u.size)
        st = self.lib.ref_step_semidiscrete(u.ctypes.data, u.size, int(periodic), origin, n_space, tau, drift,
                                            pot["kind"], pot["value"], pot["offset"], pot["amplitude"],
                                            pot["frequency"], pot["tmod"], pot["omega"], t, q, out.ctypes.data)
        return out, st

    # ---- weak-KAM consumers (proj/src/weakkam.cpp) ----
    def minplus_product(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        c = np.empty_like(a)
        st = self.lib.ref_minplus_product(a.ctypes.data, b.ctypes.data, a.shape[0], c.ctypes.data)
        if st:
            raise RuntimeError(self.err())
        return c

    def minplus_apply(self, cm, u):
        cm = np.ascontiguousarray(cm, np.float64)
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty_like(u)
        st = self.lib.ref_minplus_apply(cm.ctypes.data, cm.shape[0], u.ctypes.data, out.ctypes.data)
        if st:
            raise RuntimeError(self.err())
        return out

    def karp(self, cm):
        cm = np.ascontiguousarray(cm, np.float64)
        lam = c_double()
        st = self.lib.ref_eigenvalue_karp(cm.ctypes.data, cm.shape[0], ctypes.byref(lam))
        return lam.value, st

    @staticmethod
    def _tabs(vtabs):
        if vtabs is None:
            return None, 0
        v = np.ascontiguousarray(np.atleast_2d(vtabs), np.float64)
        return v, v.shape[0]

    def period_matrix(self, n, tau, drift, vtabs=None):
        v, nt = self._tabs(vtabs)
        c = np.empty((n, n))
        st = self.lib.ref_build_period_matrix(n, tau, drift, None if v is None else v.ctypes.data, nt,
                                              c.ctypes.data)
        if st:
            raise RuntimeError(self.err())
        return c

    def hbar_drift(self, u0, tau, drift, vtabs=None, max_periods=100, tol=1e-10):
        u0 = np.ascontiguousarray(u0, np.float64)
        v, nt = self._tabs(vtabs)
        hb, res, ns, cv = c_double(), c_double(), c_int64(), c_int()
        st = self.lib.ref_estimate_hbar_drift(u0.ctypes.data, u0.size, tau, drift,
                                              None if v is None else v.ctypes.data, nt, max_periods, tol,
                                              ctypes.byref(hb), ctypes.byref(res), ctypes.byref(ns),
                                              ctypes.byref(cv))
        return {"h_bar": hb.value, "residual": res.value, "n_steps": ns.value, "converged": bool(cv.value),
                "status": st}

    def fixed_point_residual(self, u, tau, drift, h_bar, vtabs=None):
        u = np.ascontiguousarray(u, np.float64)
        v, nt = self._tabs(vtabs)
        r = c_double()
        st = self.lib.ref_fixed_point_residual(u.ctypes.data, u.size, tau, drift,
                                               None if v is None else v.ctypes.data, nt, h_bar, ctypes.byref(r))
        return r.value, st


_ORC = None


def oracle():
    global _ORC
    if _ORC is None:
        if not os.path.exists(ORACLE_SO):
            _build_oracle()
        _ORC = Oracle(ctypes.CDLL(ORACLE_SO))
    return _ORC


def reference():
    if not os.path.exists(REF_SO) and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-f", os.path.join(ROOT, "oracle", "Makefile"), "ref"], check=True, cwd=ROOT)
    if not os.path.exists(REF_SO):
        return None
    return Reference(ctypes.CDLL(REF_SO))
