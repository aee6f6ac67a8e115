"""Solver experiments on the device: the paper's iteration-count runs.

Mirror of the Cartesian part of `dgmg.bench` (`pkg/src/dgmg/bench.py`): the
manufactured problem (three normalised Gaussian bells, `bench.py:38-90`), the
experiment configuration with the reference's defaults and consistency
rules (`bench.py:93-167`), and `run_experiment` — right-hand side, V-cycle
preconditioner, CG or GMRES to a relative residual reduction, one record per
level (`bench.py:190-300`).  Every vector lives on the device: the load
vector (`dgop.compute_rhs`), the V-cycle (`multigrid.VCycle`) and the Krylov
iteration (`krylov.pcg` / `krylov.pgmres`).  Distorted meshes
(`mesh_kind="distorted"`) run the multilinear operator,
load vector and surrogate cell smoothers of `distorted.py`.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import dgop, mesh
from .basis import Basis1D
from .krylov import pcg, pgmres
from .multigrid import MultigridConfig, VCycle
from .smoothers import SmootherConfig

__all__ = ["ManufacturedProblem", "manufactured", "ExperimentConfig", "RunRecord",
           "run_experiment"]

SIGMA = 1.0 / 3.0
BELL_CENTRES_3D = np.array([[0.0, 0.0, 0.0], [0.25, 0.85, 0.85], [0.6, 0.4, 0.4]])


@dataclass(frozen=True)
class ManufacturedProblem:
    """u = c sum_i exp(-|x - x_i|^2 / sigma^2), c = 1/(sqrt(2 pi) sigma);
    f = -Laplace u; g = u on the boundary (`bench.py:47-82`)."""

    dim: int
    sigma: float
    points: np.ndarray

    def _bells(self, x):
        x = np.atleast_2d(x)
        for p in self.points:
            r2 = ((x - p) ** 2).sum(axis=1)
            yield r2, np.exp(-r2 / self.sigma ** 2)

    def u(self, x: np.ndarray) -> np.ndarray:
        c = 1.0 / (np.sqrt(2.0 * np.pi) * self.sigma)
        out = np.zeros(len(np.atleast_2d(x)))
        for _, e in self._bells(x):
            out += e
        return c * out

    def f(self, x: np.ndarray) -> np.ndarray:
        s2 = self.sigma ** 2
        c = 1.0 / (np.sqrt(2.0 * np.pi) * self.sigma)
        out = np.zeros(len(np.atleast_2d(x)))
        for r2, e in self._bells(x):
            out += (2.0 * self.dim / s2 - 4.0 * r2 / s2 ** 2) * e
        return c * out

    def g(self, x: np.ndarray) -> np.ndarray:
        return self.u(x)


def manufactured(dim: int) -> ManufacturedProblem:
    if dim not in (2, 3):
        raise ValueError("dim must be 2 or 3")
    return ManufacturedProblem(dim=dim, sigma=SIGMA, points=BELL_CENTRES_3D[:, :dim].copy())


_OMEGA = {("acs", "cartesian"): 0.7, ("mcs", "cartesian"): 1.0, ("avs", "cartesian"): 0.25,
          ("mvs", "cartesian"): 1.0, ("acs", "distorted"): 0.5, ("mcs", "distorted"): 0.75,
          ("avs", "distorted"): 0.25, ("mvs", "distorted"): 1.0}  # bench.py:93-102


@dataclass
class ExperimentConfig:
    """`bench.py:105-167`."""

    dim: int = 2
    degree: int = 3
    coarse_cells: int | None = None
    level_min: int = 3
    level_max: int = 3
    mesh_kind: str = "cartesian"       # "cartesian" | "distorted"
    distortion: float = 0.25
    seed: int = 1234
    gamma_hat: float | None = None
    smoother: str = "acs"
    omega: float | None = None
    m_pre: int = 1
    m_post: int = 1
    solver: str | None = None          # "cg" | "gmres"
    delta_red: float = 1e-8
    symmetrize: bool | None = None
    coarse_solver: str = "auto"
    max_it: int = 200

    def resolved(self) -> "ExperimentConfig":
        cfg = replace(self)
        if cfg.dim not in (2, 3):
            raise ValueError("dim must be 2 or 3")
        if cfg.mesh_kind not in ("cartesian", "distorted"):
            raise ValueError("mesh must be cartesian or distorted")
        if cfg.smoother not in ("acs", "mcs", "avs", "mvs"):
            raise ValueError("smoother must be one of acs, mcs, avs, mvs")
        if cfg.level_min > cfg.level_max or cfg.level_min < 0:
            raise ValueError("invalid level range")
        dist = cfg.mesh_kind == "distorted"
        if cfg.coarse_cells is None:
            cfg.coarse_cells = 2 if not dist else (32 if cfg.dim == 2 else 8)
        if cfg.gamma_hat is None:
            cfg.gamma_hat = 1.0 if not dist else 4.0
        if cfg.omega is None:
            cfg.omega = _OMEGA[(cfg.smoother, cfg.mesh_kind)]
        multiplicative = cfg.smoother in ("mcs", "mvs")
        if cfg.solver is None:
            cfg.solver = "gmres" if multiplicative and not dist else "cg"
        if cfg.solver not in ("cg", "gmres"):
            raise ValueError("solver must be cg or gmres")
        if cfg.symmetrize is None:
            cfg.symmetrize = bool(multiplicative and cfg.solver == "cg")
        if multiplicative and cfg.solver == "cg" and not cfg.symmetrize:
            raise ValueError("multiplicative smoothing inside CG requires the symmetrized V-cycle")
        if dist and cfg.smoother in ("avs", "mvs"):
            raise ValueError("vertex-patch smoothers are not supported on distorted meshes")
        return cfg


@dataclass
class RunRecord:
    config: dict
    level: int
    dofs_per_level: list
    converged: bool
    iterations: int
    nu_frac: float
    wall_time: float
    ncells: int

    @property
    def dofs(self) -> int:
        return self.dofs_per_level[-1]


def _run_level(cfg: ExperimentConfig, level: int, problem: ManufacturedProblem) -> RunRecord:
    t0 = time.perf_counter()
    hier = mesh.build_hierarchy(cfg.dim, cfg.coarse_cells, level)
    basis = Basis1D.make(cfg.degree)
    dist = cfg.mesh_kind == "distorted"
    if dist:
        from . import distorted
        hier = distorted.distort(hier, cfg.distortion, cfg.seed)
        ctxs = [distorted.DistortedContext(lvl, basis, cfg.gamma_hat) for lvl in hier.levels]
    else:
        ctxs = [dgop.make_context(lvl, basis, gamma_hat=cfg.gamma_hat) for lvl in hier.levels]
    sm = SmootherConfig(kind=cfg.smoother, omega=cfg.omega, m_pre=cfg.m_pre,
                        m_post=cfg.m_post, symmetrize=cfg.symmetrize)
    cycle = VCycle(ctxs, basis, MultigridConfig(smoother=sm, coarse=cfg.coarse_solver))
    ctx = ctxs[-1]
    rhs_fn = distorted.compute_rhs if dist else dgop.compute_rhs
    apply_fn = distorted.apply_operator if dist else dgop.apply_operator
    b = torch.from_numpy(rhs_fn(ctx, problem.f, problem.g)).cuda()

    def op(x, out):
        apply_fn(ctx, x, out=out)

    def pre(r, out):
        cycle.apply(r, out)

    solve = pcg if cfg.solver == "cg" else pgmres
    res = solve(op, b, pre, delta_red=cfg.delta_red, max_it=cfg.max_it)
    torch.cuda.synchronize()
    return RunRecord(config={k: getattr(cfg, k) for k in cfg.__dataclass_fields__},
                     level=level, dofs_per_level=[c.ndofs for c in ctxs],
                     converged=res.converged, iterations=res.iterations,
                     nu_frac=res.nu_frac, wall_time=time.perf_counter() - t0,
                     ncells=ctx.layout.ncells)


def run_experiment(config: ExperimentConfig) -> list:
    """One solve of the manufactured problem per level (`bench.py:290-300`)."""
    cfg = config.resolved()
    problem = manufactured(cfg.dim)
    return [_run_level(cfg, lv, problem) for lv in range(cfg.level_min, cfg.level_max + 1)]
