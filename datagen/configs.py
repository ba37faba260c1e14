"""The five BASELINE.json workloads as concrete synthetic-input recipes.

Pure data: generator specs plus the path settings each config fits. The paper measures only
on simulated data (§6.1, L1137-1149 §6.3), so no public dataset is stood in
for. Unstated items take the readings listed in DESIGN.md §3.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import (DG_AR1, DG_BETA_ACTIVE_GROUPS, DG_BETA_EXPLICIT, DG_BETA_NORMAL, DG_BETA_UNIFORM,
               DG_BLOCK, DG_IID, DG_LINEAR, DG_LOGISTIC, DG_SPARSE, Spec, make_spec)


@dataclass
class Config:
    name: str
    spec: Spec
    penalties: list            # [(family, gamma, alpha)]
    nlambda: int
    ratio: float = 1e-3
    folds: int = 0             # K > 0: fold-segmented Gram + complements (fast CV)
    logistic: bool = False
    group_size: int = 0        # contiguous groups (cfg4)
    explicit_beta: list | None = None
    notes: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def n(self):
        return self.spec.n

    @property
    def p(self):
        return self.spec.p

    def with_n(self, n: int) -> "Config":
        """Same design and path settings at a different n (parity-size variants)."""
        return Config(self.name + f"@n={n}", self.spec.replace(n=n), self.penalties, self.nlambda,
                      self.ratio, self.folds, self.logistic, self.group_size, self.explicit_beta,
                      self.notes, dict(self.extra))


CFG1 = Config(
    "cfg1", make_spec(1, 1000, 20, DG_IID, sigma=1.0, beta_kind=DG_BETA_EXPLICIT),
    [("lasso", 0.0, 1.0)], 100,
    explicit_beta=[1.0, -1.0, 0.5, -0.5, 2.0] + [0.0] * 15,
    notes="Tiny lasso: n=1000, p=20, X iid N(0,1), beta=(1,-1,.5,-.5,2,0x15), sd 1, seed 1")

CFG2 = Config(
    "cfg2", make_spec(2, 1_000_000, 100, DG_AR1, rho=0.5, sigma=2.0, beta_kind=DG_BETA_UNIFORM,
                      nnz=10, beta_lo=-2.0, beta_hi=2.0),
    [("lasso", 0.0, 1.0), ("mcp", 3.0, 1.0), ("scad", 3.7, 1.0)], 100,
    notes="n=1e6, p=100, AR(1) rho=.5, 10 nonzero U(-2,2), sd 2; lasso+MCP(3)+SCAD(3.7), 100 lambda")

CFG3 = Config(
    "cfg3", make_spec(3, 10_000_000, 500, DG_AR1, rho=0.3, sigma=1.0, beta_kind=DG_BETA_NORMAL,
                      nnz=25),
    [("lasso", 0.0, 1.0)], 100, folds=10,
    notes="n=1e7, p=500, AR(1) rho=.3, 25 nonzero N(0,1), sd 1; 10-fold CV (i mod 10), lasso 100 lambda")

CFG4 = Config(
    "cfg4", make_spec(4, 10_000_000, 1000, DG_BLOCK, rho=0.4, group_size=10, sigma=1.0,
                      beta_kind=DG_BETA_ACTIVE_GROUPS, nnz=5),
    [("grp_lasso", 0.0, 1.0), ("enet", 0.0, 0.5)], 50, group_size=10,
    notes="n=1e7, p=1000, 100 groups of 10 with within-group corr .4, 5 active groups, sd 1; "
          "group lasso + EN(.5), 50 lambda")

CFG5 = Config(
    "cfg5", make_spec(5, 5_000_000, 200, DG_AR1, rho=0.5, response=DG_LOGISTIC,
                      beta_kind=DG_BETA_UNIFORM, nnz=20, beta_lo=-1.0, beta_hi=1.0),
    [("lasso", 0.0, 1.0)], 50, logistic=True,
    notes="Logistic n=5e6, p=200, AR(1) rho=.5, 20 nonzero U(-1,1), exact-Hessian proximal Newton, "
          "lasso 50 lambda")

# f4: the paper's sparse-design example (rsparsematrix(n, 200,
# density = 0.01), 15 nonzero coefficients U(-0.25, 0.25), noise sd 3, lasso and group lasso with
# 40 groups of 5) at the tall size of the survey's f4 row (n = 1e7; the paper used n = 1e5).
# Not one of BASELINE.json's configs: a widening of the hot path, benched as its own workload.
SPARSE = Config(
    "sparse", make_spec(6, 10_000_000, 200, DG_SPARSE, rho=0.01, sigma=3.0, beta_kind=DG_BETA_UNIFORM,
                        nnz=15, beta_lo=-0.25, beta_hi=0.25),
    [("lasso", 0.0, 1.0), ("grp_lasso", 0.0, 1.0)], 100, group_size=5,
    notes="sparse CSR design n=1e7, p=200, density 0.01 (paper §5.8 example shape), 15 nonzero "
          "U(-.25,.25), sd 3; lasso + group lasso (40 groups of 5), 100 lambda")

CONFIGS = {c.name: c for c in (CFG1, CFG2, CFG3, CFG4, CFG5, SPARSE)}


def groups_of(cfg: Config):
    """Contiguous group ids for grouped configs (cfg4: 100 groups of 10), else None."""
    import numpy as np
    if not cfg.group_size:
        return None
    return (np.arange(cfg.p) // cfg.group_size).astype(np.int32)
