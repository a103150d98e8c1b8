"""Shared fixtures for the parity tests: constant-coefficient patch problems
(the reference's const_coeffs fixture, proj/tests/test_microsim.cpp:18-30) and
small engine descriptors that both the CPU oracle and the device engine take."""
from __future__ import annotations

import numpy as np

from oracle.pyoracle import engine_desc_from_tables
from paper_2405_08764_b200 import abi, configs


def const_coef(n1, n2, A, C, Vx=0.0, Vy=0.0, W=0.0, B=0.0):
    co = np.zeros((6, n1, n2))
    co[abi.PD_COEF_A], co[abi.PD_COEF_B], co[abi.PD_COEF_C] = A, B, C
    co[abi.PD_COEF_VX], co[abi.PD_COEF_VY], co[abi.PD_COEF_W] = Vx, Vy, W
    return co


def patch_desc(coef, nx, ny, nt, h_xi, h_eta, tau, npatch=1, bc=abi.PD_BC_NEUMANN, mode=abi.PD_MODE_EXACT,
               quadrature=abi.PD_QUAD_TRAPEZOID, src_spatial=None):
    """A descriptor whose engine only serves pd_integrate_batch / lift / restrict
    (the coarse grid is a dummy row of `npatch` interior patches)."""
    d = configs.default_desc()
    d.N_xi, d.N_eta = npatch + 1, 2
    d.nx, d.ny, d.nt = nx, ny, nt
    d.k = 0
    d.tau = tau
    d.Nt, d.T = 1, 10.0 * tau
    d.h_xi, d.h_eta = h_xi, h_eta
    d.bc_type, d.quadrature = bc, quadrature
    pij = np.array([(i, 1) for i in range(1, npatch + 1)], dtype=np.int32)
    coef = np.asarray(coef, dtype=np.float64)
    if coef.ndim == 3:
        coef = np.broadcast_to(coef, (npatch,) + coef.shape).copy()
    ed = engine_desc_from_tables(d, False, (0.0, float(npatch + 1), 0.0, 2.0), pij, coef, mode=mode)
    if src_spatial is not None:
        sp = np.ascontiguousarray(np.broadcast_to(src_spatial, (npatch, nx + 1, ny + 1)), dtype=np.float64)
        ed._keep["src"] = sp
        ed.source_kind = abi.PD_SOURCE_SEPARABLE
        ed.source_spatial = sp.ctypes.data_as(type(ed.coeffs))
    return ed


def edges(kinds, n1, n2, values=None, slopes=None):
    L = max(n1, n2)
    v = np.zeros((4, L)) if values is None else np.asarray(values, dtype=np.float64)
    s = np.zeros((4, L)) if slopes is None else np.asarray(slopes, dtype=np.float64)
    return np.asarray(kinds, dtype=np.int32), v, s


N_, D_, R_ = abi.PD_EDGE_NEUMANN, abi.PD_EDGE_DIRICHLET, abi.PD_EDGE_ROBIN


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))
