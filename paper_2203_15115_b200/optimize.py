"""Augmented-Lagrangian topological level-set optimizer (SPEC ``auglag_driver``
and ``level_set_topology.fixed_point``; the reference ships no code for them,
SURVEY §0.1). Host scalar logic over device analyses.

Semantics follow ``/root/reference/SPEC.md``:
  * constraints and normalisation g:  upper g = q/(a q0) - 1,
    lower g = 1 - q/(a q0);
  * L_i (Eq 3.9), multipliers (Eq 3.11),
    penalties (Eq 3.12);
  * run (Fig 7): baseline analyses on the full domain fix q0;
    each outer step traces the volume down by dv with a fixed-point
    FEA -> fields -> combine -> extract loop; a step whose
    result violates a HARD constraint (g > 1e-6) is rejected, the last
    accepted topology restored and dv halved; the run ends when dv < dv_min;
    dv grows x1.1 (capped at dv0) after 3 consecutive accepted steps;
    multipliers/penalties update on accepted iterates only.

Builder decisions (documented in DESIGN.md §6):
  * ``displacement`` constraints (BASELINE C5: |u_z(load point)| <= 1.5x) are
    not in the SPEC's list; they are evaluated as |u_dof| and their field is
    the mutual-energy form 4/(1+nu) s(u):e(l) - (1-3nu)/(1-nu^2) tr s tr e with
    K l = e_dof (the same topological-derivative form as Eq 3.3);
  * p-norm constraints use the p of their ConstraintSpec (C4/C5: p = 8);
  * eigenvalue / buckling constraints (lower sense by default)
    run eigen.solve_modal / eigen.solve_buckling on the constrained case's
    operator; their fields are T_lambda / T_p; a buckling
    factor reported as the +inf sentinel gives g = -1.
"""

from __future__ import annotations

import logging
import math
from dataclasses import dataclass

import numpy as np

from .elements import Material
from .errors import ConfigRejected, MissingAnalysis, SemanticError
from .mesh import EPS_VOID, Domain, LoadCase, Topology, assemble_force, dirichlet_dofs

log = logging.getLogger(__name__)

KINDS = ("compliance", "pnorm_stress", "displacement", "eigenvalue", "buckling")


@dataclass(frozen=True)
class ConstraintSpec:
    """One performance constraint g_i."""

    kind: str
    alpha: float
    sense: str | None = None  # default: upper for compliance/stress/displacement, lower for eigenvalue/buckling
    soft: bool = False
    load_case: str = ""
    p: int = 6
    dof: int | None = None
    override: bool = False
    modes: int = 1            # eigenpairs computed for an eigenvalue constraint (the lowest is constrained)

    def __post_init__(self):
        if self.kind not in KINDS:
            raise SemanticError(f"unknown constraint kind {self.kind!r}")
        if self.sense is None:  # eigenvalue/buckling are lower-sense
            object.__setattr__(self, "sense", "lower" if self.kind in ("eigenvalue", "buckling") else "upper")
        if self.modes < 1:
            raise SemanticError("modes must be >= 1")
        if self.sense not in ("upper", "lower"):
            raise SemanticError(f"sense must be upper|lower, got {self.sense!r}")
        if self.sense == "lower" and not self.soft and self.alpha >= 1.0 and not self.override:
            raise ConfigRejected("a hard lower-sense constraint with alpha >= 1 is violated by the full domain: "
                                 "the algorithm will terminate at the first iteration (PAPER §3.8)")
        if self.kind == "pnorm_stress" and (self.p < 2 or self.p % 2):
            raise SemanticError("p-norm exponent must be an even integer >= 2")


@dataclass
class OptimizerConfig:
    """SPEC.md:191-194 defaults."""

    mu0: float = 100.0
    gamma0: float = 10.0
    varsigma: float = 0.25
    eta: float = 10.0
    dv0: float = 0.025
    dv_min: float = 0.005
    dv_growth: float = 1.1
    growth_after: int = 3
    inner_cap: int = 10
    compliance_tol: float = 0.01
    topology_tol: float = 0.001
    feas_tol: float = 1e-6
    ersatz: float = EPS_VOID
    tol: float = 1e-8
    eigen_tol: float = 1e-6
    block: int = 4
    max_outer: int = 400
    min_volume: float = 0.0


@dataclass
class Problem:
    domain: Domain
    material: Material
    load_cases: list
    constraints: list
    casting: object = None  # levelset.CastingSpec (PAPER §3.7) or None


@dataclass
class IterationRecord:
    k: int
    v: float
    dv: float
    accepted: bool
    q: dict
    q_over_q0: dict
    g: dict
    mu: dict
    gamma: dict
    hard_violated: bool
    J: float
    inner_iters: int
    solves: int = 0


# ---------------------------------------------------------------------------
# scalar machinery
# ---------------------------------------------------------------------------
def constraint_value(q: float, q0: float, alpha: float, sense: str) -> float:
    """SPEC.md:469. A buckling factor reported as the +inf sentinel (no
    positive factor) satisfies a lower bound: g = -1 (builder
    decision); so does any constraint whose baseline q0 is +inf (vacuous)."""
    if math.isinf(q) or math.isinf(q0):
        if sense == "lower" and q > 0.0:
            return -1.0
        if math.isinf(q0):
            return -1.0
    return q / (alpha * q0) - 1.0 if sense == "upper" else 1.0 - q / (alpha * q0)


def auglag_term(g: float, mu: float, gamma: float) -> float:
    """Eq 3.9 as printed: mu g + gamma g^2 / 2 if mu + gamma g > 0 else mu^2 / (2 gamma)."""
    if not gamma > 0.0:
        raise ValueError("penalty must be positive")
    return mu * g + 0.5 * gamma * g * g if mu + gamma * g > 0.0 else 0.5 * mu * mu / gamma


def update_multiplier(mu: float, gamma: float, g: float) -> float:
    """Eq 3.11."""
    return max(mu + gamma * g, 0.0)


def update_penalty(gamma: float, g_prev: float, g_new: float, k: int, varsigma: float = 0.25,
                   eta: float = 10.0) -> float:
    """Eq 3.12."""
    if min(g_new, 0.0) <= varsigma * min(g_prev, 0.0):
        return gamma
    return max(eta * gamma, float(k * k))


def evaluate_constraints(specs, q: dict, q0: dict) -> dict:
    """g per constraint name; raises MissingAnalysis if a quantity is absent."""
    out = {}
    for name, spec in specs.items():
        if name not in q or name not in q0:
            raise MissingAnalysis(f"constraint {name!r} has no analysis")
        out[name] = constraint_value(q[name], q0[name], spec.alpha, spec.sense)
    return out


# ---------------------------------------------------------------------------
# device analyses
# ---------------------------------------------------------------------------
def _case_data(problem: Problem, case):
    """(sorted fixed DOFs, device force vector) of a load case. They depend on
    the domain and the case only, so they are built once per problem (the
    host-side selector evaluation over all nodes costs ~0.1 s at C4)."""
    cache = problem.__dict__.setdefault("_case_cache", {})
    if case.id not in cache:
        torch = __import__("torch")
        cache[case.id] = (dirichlet_dofs(problem.domain, case),
                          torch.from_numpy(assemble_force(problem.domain, case)).cuda())
    return cache[case.id]


class Analyses:
    """FEA + sensitivity fields of one topology for every load case (device)."""

    def __init__(self, problem: Problem, specs: dict, topology: Topology, cfg: OptimizerConfig, need_fields=True):
        from . import fea, sensitivity

        torch = __import__("torch")
        self.topology = topology
        d = problem.domain
        self.q = {}
        self.fields = {}
        self.J = {}
        self.solves = 0
        cases = {c.id: c for c in problem.load_cases}
        for name, spec in specs.items():
            if spec.load_case not in ("", *cases):
                raise MissingAnalysis(f"constraint {name!r} refers to unknown load case {spec.load_case!r}")
            if spec.kind == "displacement" and spec.dof is None:
                raise SemanticError(f"displacement constraint {name!r} needs a dof")
        # load cases sharing a Dirichlet set share one operator / deflation
        # space and are solved together (multi-RHS batch, fea.solve_static_batch);
        # so are their adjoint right-hand sides
        groups = {}
        for case in problem.load_cases:
            fixed, f = _case_data(problem, case)
            key = fixed.tobytes()
            if key not in groups:
                op = fea.StiffnessOperator(d, topology, problem.material, fixed)
                defl = fea.build_deflation(d, topology, fixed, cfg.block) if cfg.block else None
                groups[key] = (op, defl, [])
            groups[key][2].append((case, f))
        for op, defl, members in groups.values():
            sols = fea.solve_static_batch(op, [f for _, f in members], tol=cfg.tol, deflation=defl)
            self.solves += len(members)
            adjoints = []  # (constraint name, u, adjoint rhs)
            for (case, f), sol in zip(members, sols):
                u = sol.u
                self.J[case.id] = float(f @ u)
                vm, tj, _ = sensitivity.element_fields_device(op, u, 2)
                for name, spec in specs.items():
                    if (spec.load_case or problem.load_cases[0].id) != case.id:
                        continue
                    if spec.kind == "compliance":
                        self.q[name] = self.J[case.id]
                        if need_fields:
                            self.fields[name] = tj
                    elif spec.kind == "pnorm_stress":
                        _, _, sums = sensitivity.element_fields_device(op, u, spec.p)
                        s = sums.cpu().numpy()
                        self.q[name] = float((s[0] / s[1]) ** (1.0 / spec.p))
                        if need_fields:
                            adjoints.append((name, u, sensitivity.adjoint_rhs_device(op, u, spec.p, sums)))
                    elif spec.kind == "displacement":
                        self.q[name] = abs(float(u[spec.dof]))
                        if need_fields:
                            e = torch.zeros_like(u)
                            e[spec.dof] = math.copysign(1.0, float(u[spec.dof]))
                            adjoints.append((name, u, e))
            self._eigen_analyses(problem, specs, cfg, op, defl, members, sols, need_fields)
            if adjoints:
                lams = fea.solve_static_batch(op, [rhs for _, _, rhs in adjoints], tol=cfg.tol, deflation=defl)
                self.solves += len(adjoints)
                for (name, u, _), lam in zip(adjoints, lams):
                    self.fields[name] = sensitivity.stress_sensitivity(op, u, lam.u)
        self.J_total = float(sum(self.J.values()))

    def _eigen_analyses(self, problem, specs, cfg, op, defl, members, sols, need_fields):
        """Modal and buckling analyses of
        the constraints attached to this Dirichlet group; only run when a
        constraint asks for them."""
        from . import eigen

        torch = __import__("torch")
        ids = {case.id: i for i, (case, _) in enumerate(members)}
        modal = None
        for name, spec in specs.items():
            cid = spec.load_case or problem.load_cases[0].id
            if cid not in ids:
                continue
            if spec.kind == "eigenvalue":
                if modal is None or len(modal.values) < spec.modes:
                    modal = eigen.solve_modal(op, eigen.MassOperator(op), k=spec.modes, tol=cfg.eigen_tol,
                                              deflation=defl)
                    self.solves += modal.solves
                self.q[name] = float(modal.values[0])
                if need_fields:
                    self.fields[name] = eigen.eigen_sensitivity(op, modal.vectors[0], modal.values[0])
            elif spec.kind == "buckling":
                u = sols[ids[cid]].u
                geo = eigen.geometric_stiffness(u, op)
                r = eigen.solve_buckling(op, geo, k=1, tol=cfg.eigen_tol, deflation=defl)
                self.solves += r.solves
                self.q[name] = float(r.values[0])
                if need_fields:
                    self.fields[name] = (torch.zeros(op.domain.n_elems, dtype=torch.float64, device="cuda")
                                         if r.no_positive_factor else
                                         eigen.buckling_sensitivity(op, geo, r.vectors[0], r.values[0]))


def _compliance_fallback(specs: dict) -> str:
    for name, spec in specs.items():
        if spec.kind == "compliance":
            return name
    return next(iter(specs))


def fixed_point(problem: Problem, specs: dict, start: Analyses, target_vf: float, weights: dict,
                cfg: OptimizerConfig):
    """iterate FEA -> fields -> combine -> extract at the
    target fraction. Returns (Analyses, converged, inner_iterations, solves)."""
    from .levelset import combine_device, extract_device

    torch = __import__("torch")
    names = list(specs)
    fallback = _compliance_fallback(specs)
    design = torch.from_numpy(problem.domain.design_mask.astype(np.uint8)).cuda()
    cur = start
    prev_occ = start.topology.occupancy
    solves = 0
    for it in range(1, cfg.inner_cap + 1):
        w = [weights[n] for n in names]
        if all(x == 0.0 for x in w):
            ls = combine_device([cur.fields[fallback]], [1.0])
        else:
            keep = [(cur.fields[n], x) for n, x in zip(names, w) if x != 0.0]
            ls = combine_device([k for k, _ in keep], [x for _, x in keep])
        occ_d, _, _ = extract_device(problem.domain, ls, target_vf, cfg.ersatz, design, casting=problem.casting)
        occ = occ_d.cpu().numpy()
        changed = int(np.count_nonzero((occ == 1.0) != (prev_occ == 1.0)))
        if it > 1 and changed < cfg.topology_tol * problem.domain.n_elems:
            return cur, True, it, solves
        nxt = Analyses(problem, specs, Topology(problem.domain, occ), cfg)
        solves += nxt.solves
        if it > 1 and abs(nxt.J_total - cur.J_total) < cfg.compliance_tol * cur.J_total:
            return nxt, True, it, solves
        cur, prev_occ = nxt, occ
    return cur, False, cfg.inner_cap, solves


def run(problem: Problem, config: OptimizerConfig | None = None, callback=None):
    """Fig 7 / SPEC.md:237-246. Returns (topology, history, reason)."""
    cfg = config or OptimizerConfig()
    if not (0.0 < cfg.varsigma < 1.0 and cfg.eta > 0.0 and 0.0 < cfg.dv_min <= cfg.dv0 < 1.0):
        raise SemanticError("invalid optimizer configuration")
    if not problem.constraints:
        raise SemanticError("at least one constraint is required")
    specs = {f"{c.kind}:{c.load_case or problem.load_cases[0].id}:{i}": c for i, c in enumerate(problem.constraints)}
    d = problem.domain
    full = Topology(d)
    base = Analyses(problem, specs, full, cfg)
    q0 = dict(base.q)
    g = evaluate_constraints(specs, base.q, q0)
    mu = {n: cfg.mu0 for n in specs}
    gamma = {n: cfg.gamma0 for n in specs}
    accepted = base
    dv = cfg.dv0
    streak = 0
    history = []
    reason = "max_outer"
    total_solves = base.solves
    for k in range(1, cfg.max_outer + 1):
        v = accepted.topology.volume_fraction
        target = v - dv
        if target <= max(cfg.min_volume, 1.0 / d.n_design):
            reason = "minimum volume reached"
            break
        weights = {n: max(mu[n] + gamma[n] * g[n], 0.0) for n in specs}
        res, conv, inner, solves = fixed_point(problem, specs, accepted, target, weights, cfg)
        total_solves += solves
        g_new = evaluate_constraints(specs, res.q, q0)
        hard = any((not specs[n].soft) and g_new[n] > cfg.feas_tol for n in specs)
        rec = IterationRecord(k=k, v=res.topology.volume_fraction, dv=dv, accepted=not hard, q=dict(res.q),
                              q_over_q0={n: res.q[n] / q0[n] for n in specs}, g=dict(g_new), mu=dict(mu),
                              gamma=dict(gamma), hard_violated=hard, J=res.J_total, inner_iters=inner,
                              solves=solves)
        history.append(rec)
        if callback:
            callback(rec)
        if hard:
            dv *= 0.5
            streak = 0
            if dv < cfg.dv_min:
                reason = "volume step below dv_min with a hard constraint violated"
                break
            continue
        for n in specs:
            new_mu = update_multiplier(mu[n], gamma[n], g_new[n])
            gamma[n] = update_penalty(gamma[n], g[n], g_new[n], k, cfg.varsigma, cfg.eta)
            mu[n] = new_mu
        g = g_new
        accepted = res
        streak += 1
        if streak >= cfg.growth_after:
            dv = min(dv * cfg.dv_growth, cfg.dv0)
    log.info("optimizer stopped after %d outer steps (%d solves): %s", len(history), total_solves, reason)
    return accepted.topology, history, reason


def cantilever_problem(nx, ny, nz, load_min, load_max, force=(0.0, 0.0, -1.0), E=1.0, nu=0.3,
                       constraints=None, extra_cases=()):
    """Convenience builder of the BASELINE cantilever configs."""
    from .mesh import RegionSelector

    d = Domain(nx, ny, nz, 1.0)
    clamp = ((RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),)
    cases = [LoadCase("load", dirichlet=clamp, loads=((RegionSelector("box", min=load_min, max=load_max), force,
                                                        "total"),))]
    for cid, lo, hi, fv in extra_cases:
        cases.append(LoadCase(cid, dirichlet=clamp, loads=((RegionSelector("box", min=lo, max=hi), fv, "total"),)))
    if constraints is None:
        constraints = [ConstraintSpec("compliance", 1.6)]
    return Problem(d, Material(E=E, nu=nu), cases, list(constraints))


__all__ = [
    "ConstraintSpec", "OptimizerConfig", "Problem", "IterationRecord", "Analyses", "constraint_value",
    "auglag_term", "update_multiplier", "update_penalty", "evaluate_constraints", "fixed_point", "run",
    "cantilever_problem",
]

