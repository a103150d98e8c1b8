"""Config files (configs/*.cfg) -> pd_problem_desc.

Flat ``key = value`` lines under ``[section]`` headers, ``#`` comments, unknown
keys rejected — the reference's config conventions (proj/src/config.cpp:78-264).
Every BASELINE pin is spelled out in the files.
"""
from __future__ import annotations

import configparser
from pathlib import Path

from . import abi
from .abi import ProblemDesc

ROOT = Path(__file__).resolve().parent.parent
CONFIG_DIR = ROOT / "configs"

KINDS = {
    "diffusion-square": abi.PD_PROBLEM_DIFFUSION_SQUARE,
    "cdr-tanh": abi.PD_PROBLEM_CDR_TANH,
    "annulus-nonaxi": abi.PD_PROBLEM_ANNULUS_NONAXI,
    "shear-cdr": abi.PD_PROBLEM_SHEAR_CDR,
    "ref-annulus": abi.PD_PROBLEM_REF_ANNULUS,
    "ref-cdr": abi.PD_PROBLEM_REF_CDR,
    "ref-cdr-var": abi.PD_PROBLEM_REF_CDR_VAR,
    "steady": abi.PD_PROBLEM_STEADY,
    "pulsed-cdr": abi.PD_PROBLEM_PULSED_CDR,
}
BC = {"neumann": abi.PD_BC_NEUMANN, "dirichlet": abi.PD_BC_DIRICHLET, "robin": abi.PD_BC_ROBIN}
QUAD = {"trapezoid": abi.PD_QUAD_TRAPEZOID, "simpson": abi.PD_QUAD_SIMPSON}
DT = {"given": abi.PD_DT_GIVEN, "diffusion": abi.PD_DT_DIFFUSION, "metric": abi.PD_DT_METRIC}
MODE = {"fast": abi.PD_MODE_FAST, "exact": abi.PD_MODE_EXACT}
SOLVER = {"explicit": abi.PD_SOLVER_EXPLICIT, "adi": abi.PD_SOLVER_ADI}  # micro.solver (config.cpp:169-172)
UPWIND = {"two": abi.PD_UPWIND_TWO, "three": abi.PD_UPWIND_THREE, "four": abi.PD_UPWIND_FOUR}  # config.cpp:173-179

_SCHEMA = {
    "problem": {"kind": str, "lambda": float, "beta": float, "eps": float, "omega": float, "vel": float,
                "amp": float, "seed": int, "jacobi_sweeps": int},
    "scheme": {"n_xi": int, "n_eta": int, "nt_macro": int, "k": int, "T": float, "tau": float,
               "h_xi": float, "h_eta": float, "h_frac": float, "dt_over_tau": float},
    "micro": {"nx": int, "ny": int, "nt": int, "dt_rule": str, "bc_type": str, "robin_w1": float,
              "robin_w2": float, "quadrature": str, "mode": str, "solver": str, "upwind": str,
              "upwind_r": float},
    "sweep": {"log2_patches": str, "micro_nodes": str, "K": str},
}


def default_desc() -> ProblemDesc:
    d = ProblemDesc()
    d.eps = 1.0
    d.beta = 3.0
    d.vel = 1.0
    d.amp = 0.1
    d.seed = 20240514
    d.N_xi = d.N_eta = 10
    d.Nt = 100
    d.T = 1.0
    d.tau = 1e-6
    d.h_xi = d.h_eta = 1e-3
    d.nx = d.ny = 10
    d.nt = 2
    d.robin_w1 = d.robin_w2 = 1.0
    d.mode = abi.PD_MODE_FAST
    d.solver = abi.PD_SOLVER_EXPLICIT  # the BASELINE configs' micro-solver (the reference's default is ADI)
    d.upwind_order = abi.PD_UPWIND_TWO
    d.upwind_r = 0.5  # UpwindSpec::r default (microsim.hpp:47)
    return d


def parse(text: str, origin: str = "<config>") -> tuple[ProblemDesc, dict]:
    cp = configparser.ConfigParser(inline_comment_prefixes=("#",), comment_prefixes=("#",))
    cp.optionxform = str
    cp.read_string(text, source=origin)
    vals: dict = {}
    for sec in cp.sections():
        if sec not in _SCHEMA:
            raise ValueError(f"{origin}: unknown section [{sec}]")
        for key, raw in cp.items(sec):
            if key not in _SCHEMA[sec]:
                raise ValueError(f"{origin}: unknown key '{sec}.{key}'")
            vals[f"{sec}.{key}"] = _SCHEMA[sec][key](raw.strip())
    d = default_desc()
    kind = vals.get("problem.kind")
    if kind not in KINDS:
        raise ValueError(f"{origin}: unknown problem kind {kind!r}")
    d.problem = KINDS[kind]
    simple = {"problem.lambda": "lambda_", "problem.beta": "beta", "problem.eps": "eps", "problem.omega": "omega",
              "problem.vel": "vel", "problem.amp": "amp", "problem.seed": "seed",
              "problem.jacobi_sweeps": "jacobi_sweeps", "scheme.n_xi": "N_xi", "scheme.n_eta": "N_eta",
              "scheme.nt_macro": "Nt", "scheme.k": "k", "scheme.T": "T", "scheme.tau": "tau",
              "scheme.h_xi": "h_xi", "scheme.h_eta": "h_eta", "scheme.h_frac": "h_frac",
              "scheme.dt_over_tau": "dt_over_tau", "micro.nx": "nx", "micro.ny": "ny", "micro.nt": "nt",
              "micro.robin_w1": "robin_w1", "micro.robin_w2": "robin_w2", "micro.upwind_r": "upwind_r"}
    for k, f in simple.items():
        if k in vals:
            setattr(d, f, vals[k])
    if "micro.dt_rule" in vals:
        d.dt_rule = DT[vals["micro.dt_rule"]]
    if "micro.bc_type" in vals:
        d.bc_type = BC[vals["micro.bc_type"]]
    if "micro.quadrature" in vals:
        d.quadrature = QUAD[vals["micro.quadrature"]]
    if "micro.mode" in vals:
        d.mode = MODE[vals["micro.mode"]]
    if "micro.solver" in vals:
        d.solver = SOLVER[vals["micro.solver"]]
    if "micro.upwind" in vals:
        d.upwind_order = UPWIND[vals["micro.upwind"]]
    return d, vals


def load(name_or_path) -> tuple[ProblemDesc, dict]:
    p = Path(name_or_path)
    if not p.exists():
        p = CONFIG_DIR / (str(name_or_path) if str(name_or_path).endswith(".cfg") else f"{name_or_path}.cfg")
    return parse(p.read_text(), str(p))


def copy_desc(d: ProblemDesc, **over) -> ProblemDesc:
    n = ProblemDesc()
    for f, _ in ProblemDesc._fields_:
        setattr(n, f, getattr(d, f))
    for k, v in over.items():
        setattr(n, k, v)
    return n


def sweep_desc(base: ProblemDesc, log2_patches: int, nodes: int, K: int, **over) -> ProblemDesc:
    """Config-5 sweep point: 2^k patches (square for even k, 2:1 for odd k)."""
    k = log2_patches
    px = 2 ** ((k + 1) // 2)
    py = 2 ** (k // 2)
    return copy_desc(base, N_xi=px + 1, N_eta=py + 1, nx=nodes - 1, ny=nodes - 1, nt=K, **over)
