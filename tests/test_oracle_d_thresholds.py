"""Pins for oracle O4 (eigenvalues / d rule) and the thresholding operators of PAPER.md §2.2.

Thresholds are pinned by SPEC's printed values, by a brute-force numeric prox (each operator must
be the exact minimiser of 0.5 d b^2 - u b + P(b), P from Table 1), and by the textbook d = 1
forms (Zhang's firm threshold, Fan & Li's SCAD rule)."""
import math

import numpy as np
import pytest
from scipy.optimize import minimize, minimize_scalar

import oracle as orc


# ------------------------------------------------------------------ d
def test_eigen_examples(golden):
    """d(I_2) = 1 and d([[2,1],[1,2]]) = 3 EXACTLY: both are Gershgorin-tight
    (constant row sums of a nonnegative matrix), so the rule's min takes the Gershgorin value."""
    for ex in golden["largest_eigenvalue"]:
        A = np.array(ex["A"])
        assert abs(orc.eig_jacobi(A)[-1] - ex["lambda1"]) < 1e-15
        d, U, gs = orc.d_rule(A)
        assert d == ex["lambda1"] and gs == ex["lambda1"]
        assert U > ex["lambda1"]            # the trace bound is the looser branch here


PHI2 = (3.0 + math.sqrt(5.0)) / 2.0        # largest eigenvalue of [[2,1],[1,1]]
ALLOW = 2 * 12 * 2.0 ** -53                 # R#5 rounding allowance (1 + 2 S p u), per unit of p


def test_d_rule_trace_branch_closed_forms():
    """R#5 values by hand where the trace branch U_S is the one taken (Gershgorin = 3):
    [[2,1],[1,1]] has eigenvalues phi^2, phi^-2, so U_S = phi^2 (1 + phi^(-4 * 2^S))^(2^-S) = phi^2
    in fp64; two copies (block diagonal) double every eigenvalue's multiplicity, so
    U_S = 2^(2^-S) phi^2 -- which pins the exponent S = 12 (S = 11 or 13 differ by 1.7e-4 / 8.5e-5
    relative). A scalar multiple scales d exactly linearly."""
    A = np.array([[2.0, 1.0], [1.0, 1.0]])
    d, U, gs = orc.d_rule(A)
    assert gs == 3.0 and abs(d - PHI2 * (1 + ALLOW * 2)) <= 4e-16 * PHI2
    B = np.kron(np.eye(2), A)
    d2, U2, gs2 = orc.d_rule(B)
    assert gs2 == 3.0 and abs(d2 - PHI2 * 2.0 ** (1.0 / 4096) * (1 + ALLOW * 4)) <= 4e-16 * PHI2
    assert abs(d2 / PHI2 - 1.0 - math.log(2.0) / 4096) < 1e-7
    d7, _, _ = orc.d_rule(7.0 * B)
    assert abs(d7 - 7.0 * d2) <= 1e-15 * d7
    # p copies of one eigenvalue: U_S = c p^(2^-S) exactly, Gershgorin = c (d = c)
    for p in (1, 3, 50):
        dI, UI, gI = orc.d_rule(2.5 * np.eye(p))
        assert dI == 2.5 and abs(UI - 2.5 * p ** (1.0 / 4096) * (1 + ALLOW * p)) <= 1e-15 * UI
    # the number of squarings is an argument: S = 1 gives sqrt(trace(A^2)) = ||A||_F
    _, U1, _ = orc.d_rule(A, squarings=1)
    assert abs(U1 - math.sqrt(7.0) * (1 + 4 * 2.0 ** -53)) <= 1e-15 * U1


def test_d_rule_eigenvector_orthogonal_to_ones():
    """a rule seeded with 1/sqrt(p) under-estimated lambda_1 when the top
    eigenvector is orthogonal to the all-ones vector. The trace bound does not depend on any
    start vector: d >= lambda_1 on every such case."""
    cases = []
    cases.append(np.array([[1.0, -0.482], [-0.482, 1.0]]))        # standardized p = 2, rho < 0
    cases.append(np.eye(3) - np.full((3, 3), 1.0 / 3.0))          # centred 3-simplex (1 in the null space)
    rng = np.random.default_rng(11)
    Xpm = rng.choice([-1.0, 1.0], size=(64, 6))
    Xpm[:, 1] = -Xpm[:, 0]                                        # perfectly negatively correlated +-1 pair
    cases.append(Xpm.T @ Xpm / 64)
    D = np.eye(4)[rng.integers(0, 4, 200)]                         # one-hot dummies, centred
    D -= D.mean(axis=0)
    cases.append(D.T @ D / 200)
    for A in cases:
        lam1 = np.linalg.eigvalsh(A)[-1]
        d, U, gs = orc.d_rule(A)
        assert lam1 <= d * (1 + 1e-13)
        assert d <= lam1 * A.shape[0] ** (1.0 / 4096) * (1 + ALLOW * A.shape[0] + 1e-14)


@pytest.mark.parametrize("kind", ["ar1_0.5", "ar1_0.3", "block_0.4", "iid", "spike"])
def test_d_rule_brackets_lambda1(kind):
    """R#5: lambda_1 <= U_S <= p^(2^-S) lambda_1 (the trace inequality), so
    lambda_1 <= d <= 1.0012 lambda_1 at p = 100, with lambda_1 from cyclic Jacobi and numpy, on
    the configs' population Grams, on sample Grams of those designs, and on a spike barely above
    a 99-fold bulk (the case a 200-step Rayleigh quotient misses by 0.5%)."""
    rng = np.random.default_rng(8)
    p = 100
    if kind.startswith("ar1"):
        rho = float(kind.split("_")[1])
        S = rho ** np.abs(np.subtract.outer(np.arange(p), np.arange(p)))
    elif kind.startswith("block"):
        S = np.kron(np.eye(10), np.full((10, 10), 0.4)) + 0.6 * np.eye(p)
    elif kind == "spike":
        Q, _ = np.linalg.qr(rng.standard_normal((p, p)))
        S = Q @ np.diag(np.r_[1.0, np.full(p - 1, 0.99)]) @ Q.T
        S = (S + S.T) / 2
    else:
        S = np.eye(p)
    L = np.linalg.cholesky(S)
    for A in (S, (lambda Z: Z.T @ Z / Z.shape[0])(rng.standard_normal((4000, p)) @ L.T)):
        lam1 = np.linalg.eigvalsh(A)[-1]
        assert abs(orc.eig_jacobi(A)[-1] - lam1) <= 1e-13 * lam1
        d, U, gs = orc.d_rule(A)
        assert gs >= lam1 * (1 - 1e-12)          # Gershgorin bound
        assert U >= lam1 * (1 - 1e-13)           # trace bound
        assert U <= lam1 * p ** (1.0 / 4096) * (1 + ALLOW * p + 1e-14)
        assert d == min(gs, U)


def test_d_rule_trace_sum_matches_eigenvalues():
    """U_S^(2^S) = sum_i lambda_i^(2^S): for a matrix with a known spectrum the rule's value is
    that sum's root, computed here in logs from the eigenvalues themselves."""
    rng = np.random.default_rng(5)
    p = 12
    lam = np.sort(rng.uniform(0.5, 2.0, p))
    lam[-3:] = [1.9, 1.95, 2.0]
    Q, _ = np.linalg.qr(rng.standard_normal((p, p)))
    A = Q @ np.diag(lam) @ Q.T
    A = (A + A.T) / 2
    _, U, _ = orc.d_rule(A)
    m = 4096.0
    expect = lam[-1] * np.exp(np.log(np.sum(np.exp(m * (np.log(lam) - np.log(lam[-1]))))) / m)
    expect *= 1 + ALLOW * p
    assert abs(U - expect) <= 1e-13 * expect


# ------------------------------------------------------------------ thresholds: printed values
def test_spec_printed_values(golden):
    for ex in golden["soft"]:
        assert orc.soft(ex["u"], ex["lam"], ex["d"]) == ex["out"]
    for ex in golden["enet"]:
        assert abs(orc.enet(ex["u"], ex["lam"], ex["alpha"], ex["d"]) - ex["out"]) < 1e-15
    for ex in golden["mcp"]:
        assert orc.mcp(ex["u"], ex["lam"], ex["gamma"], ex["d"]) == ex["out"]
    for ex in golden["scad"]:
        out = ex.get("out", ex.get("out_num", 0) / ex.get("out_den", 1))
        assert abs(orc.scad(ex["u"], ex["lam"], ex["gamma"], ex["d"]) - out) < 1e-15
    for ex in golden["grp_lasso"]:
        assert np.allclose(orc.grp_lasso(ex["u"], ex["lam"], ex["d"]), ex["out"], atol=1e-15)
    for ex in golden["grp_mcp"]:
        assert np.allclose(orc.grp_mcp(ex["u"], ex["lam"], ex["gamma"], ex["d"]), ex["out"], atol=1e-15)


# ------------------------------------------------------------------ penalty forms (Table 1)
def p_mcp(b, lam, g):
    a = abs(b)
    return lam * a - a * a / (2 * g) if a <= g * lam else g * lam * lam / 2


def p_scad(b, lam, g):
    a = abs(b)
    if a <= lam:
        return lam * a
    if a <= g * lam:
        return -(a * a - 2 * g * lam * a + lam * lam) / (2 * (g - 1))
    return (g + 1) * lam * lam / 2


def numeric_prox(u, d, pen):
    """argmin_b 0.5 d b^2 - u b + pen(b): dense grid then bounded Brent refinement."""
    hi = abs(u) / d + 1.0
    grid = np.linspace(-hi, hi, 20001)
    vals = 0.5 * d * grid ** 2 - u * grid + np.array([pen(b) for b in grid])
    b0 = grid[np.argmin(vals)]
    step = grid[1] - grid[0]
    res = minimize_scalar(lambda b: 0.5 * d * b * b - u * b + pen(b), bounds=(b0 - 2 * step, b0 + 2 * step),
                          method="bounded", options={"xatol": 1e-12})
    return res.x


def test_prox_fidelity_scalar():
    """every scalar operator is the exact prox of its Table 1 penalty with divisor d."""
    rng = np.random.default_rng(9)
    for _ in range(250):
        d = rng.uniform(1.0, 4.0)
        u = rng.uniform(-6, 6)
        lam = rng.uniform(0.05, 2.0)
        alpha = rng.uniform(0.05, 1.0)
        g_m = rng.uniform(1.0 / d + 0.6, 6.0)        # gamma*d > 1 (R#8)
        g_s = rng.uniform(max(2.0, 1.0 / d + 1.0) + 0.3, 7.0)  # gamma > 2, (gamma-1)d > 1
        assert abs(orc.soft(u, lam, d) - numeric_prox(u, d, lambda b: lam * abs(b))) < 1e-6
        assert abs(orc.enet(u, lam, alpha, d) - numeric_prox(
            u, d, lambda b: alpha * lam * abs(b) + 0.5 * (1 - alpha) * lam * b * b)) < 1e-6
        assert abs(orc.mcp(u, lam, g_m, d) - numeric_prox(u, d, lambda b: p_mcp(b, lam, g_m))) < 1e-6
        assert abs(orc.scad(u, lam, g_s, d) - numeric_prox(u, d, lambda b: p_scad(b, lam, g_s))) < 1e-6


def test_textbook_forms_at_d1():
    """At d = 1: MCP = Zhang's firm threshold, SCAD = Fan & Li (2001) three-piece rule."""
    rng = np.random.default_rng(10)
    for _ in range(500):
        u, lam = rng.uniform(-8, 8), rng.uniform(0.1, 2)
        g = rng.uniform(1.5, 5)
        firm = (np.sign(u) * g * max(abs(u) - lam, 0) / (g - 1)) if abs(u) <= g * lam else u
        assert abs(orc.mcp(u, lam, g, 1.0) - firm) < 1e-14
        a = rng.uniform(2.2, 5)
        if abs(u) <= 2 * lam:
            fl = np.sign(u) * max(abs(u) - lam, 0)
        elif abs(u) <= a * lam:
            fl = ((a - 1) * u - np.sign(u) * a * lam) / (a - 2)
        else:
            fl = u
        assert abs(orc.scad(u, lam, a, 1.0) - fl) < 1e-13


def test_continuity_and_limits():
    for d in (1.0, 2.5):
        lam, g = 0.7, 3.7
        for edge in (lam, (d + 1) * lam, g * lam * d):
            for f in (lambda u: orc.scad(u, lam, g, d), lambda u: orc.mcp(u, lam, g, d),
                      lambda u: orc.soft(u, lam, d)):
                assert abs(f(edge + 1e-9) - f(edge - 1e-9)) < 1e-6
        # gamma -> infinity: MCP and SCAD -> soft threshold
        for u in np.linspace(-5, 5, 41):
            assert abs(orc.mcp(u, lam, 1e7, d) - orc.soft(u, lam, d)) < 1e-6
            assert abs(orc.scad(u, lam, 1e7, d) - orc.soft(u, lam, d)) < 1e-6


def test_group_prox_fidelity():
    """Group operators are the exact prox of c*lam*P(||b||) with divisor d."""
    rng = np.random.default_rng(11)
    for _ in range(30):
        d = rng.uniform(1.0, 3.0)
        u = rng.uniform(-3, 3, 3)
        lam = rng.uniform(0.1, 2.0)
        g = rng.uniform(1.0 / d + 1.0, 5.0)
        gs = rng.uniform(max(2.0, 1.0 / d + 1.0) + 0.5, 6.0)
        for op, pen in ((lambda: orc.grp_lasso(u, lam, d), lambda nb: lam * nb),
                        (lambda: orc.grp_mcp(u, lam, g, d), lambda nb: p_mcp(nb, lam, g)),
                        (lambda: orc.grp_scad(u, lam, gs, d), lambda nb: p_scad(nb, lam, gs))):
            f = lambda b: 0.5 * d * b @ b - u @ b + pen(np.linalg.norm(b))
            best = None
            for start in (np.zeros(3), u / d, 0.5 * u / d):
                r = minimize(f, start, method="Nelder-Mead",
                             options={"xatol": 1e-11, "fatol": 1e-15, "maxiter": 20000})
                if best is None or r.fun < best.fun:
                    best = r
            out = op()
            assert f(out) <= best.fun + 1e-10
            assert np.max(np.abs(out - best.x)) < 1e-4


def test_group_zero_norm():
    z = np.zeros(4)
    assert not orc.grp_lasso(z, 1.0, 2.0).any()
    assert not orc.grp_mcp(z, 1.0, 3.0, 2.0).any()
    assert not orc.grp_scad(z, 1.0, 3.7, 2.0).any()


# ---------------------------------------------------------------- sparse group lasso (f3, R#11)
def _sgl_objective(b, u, lam, tau, c, d, w):
    return 0.5 * d * b @ b - u @ b + lam * tau * np.sum(w * np.abs(b)) + lam * (1 - tau) * c * np.linalg.norm(b)


def test_sgl_paper_formula_at_d1():
    """At d = 1 the operator is the paper's printed composition G(v, c lam (1 - tau), 1) with
    v_j = S(u_j, w_j lam tau, 1), written out here from the equations."""
    rng = np.random.default_rng(31)
    for _ in range(200):
        m = int(rng.integers(1, 6))
        u = rng.normal(0, 2, m)
        w = rng.uniform(0.5, 2.0, m)
        lam, tau, c = rng.uniform(0.05, 1.5), rng.uniform(0, 1), rng.uniform(0.5, 3)
        v = np.sign(u) * np.maximum(np.abs(u) - w * lam * tau, 0.0)          # eq (lasso), d = 1
        nv = np.linalg.norm(v)
        g = v * max(0.0, 1 - c * lam * (1 - tau) / nv) if nv > 0 else 0 * v  # eq (glasso), d = 1
        assert np.allclose(orc.sgl(u, lam, tau, c, 1.0, w), g, rtol=0, atol=1e-15)


def test_sgl_is_the_exact_prox_at_any_d():
    """For d in {2, 3} the composed operator minimises the M-step objective
    (d/2)||b||^2 - u^T b + P_sgl(b) (numeric minimiser, Nelder-Mead from the closed form and from
    zero); the printed d = 1 composition does not (R#11)."""
    from scipy.optimize import minimize
    rng = np.random.default_rng(32)
    worse = 0
    for _ in range(60):
        m = int(rng.integers(2, 4))
        u = rng.normal(0, 3, m)
        w = rng.uniform(0.5, 1.5, m)
        lam, tau, c, d = rng.uniform(0.1, 1.0), rng.uniform(0.1, 0.9), rng.uniform(0.5, 2), float(rng.choice([2.0, 3.0]))
        b = orc.sgl(u, lam, tau, c, d, w)
        f = lambda x: _sgl_objective(x, u, lam, tau, c, d, w)  # noqa: E731
        best = min((minimize(f, x0, method="Nelder-Mead", options={"xatol": 1e-12, "fatol": 1e-14, "maxiter": 20000})
                    for x0 in (b + 1e-3, np.zeros(m), u / d)), key=lambda r: r.fun)
        assert f(b) <= best.fun + 1e-9
        v = np.sign(u) * np.maximum(np.abs(u) - w * lam * tau, 0.0) / d
        nv = np.linalg.norm(v)
        printed = v * max(0.0, 1 - c * lam * (1 - tau) / nv) if nv > 0 else 0 * v
        worse += f(printed) > f(b) + 1e-9
    assert worse > 0   # the printed d = 1 form is not the M-step minimiser in general


def test_sgl_limits():
    """tau = 0: group lasso; tau = 1: coordinate-wise lasso."""
    rng = np.random.default_rng(33)
    for _ in range(50):
        u = rng.normal(0, 2, 4)
        lam, c, d = rng.uniform(0.1, 2), rng.uniform(0.5, 2), rng.uniform(1, 3)
        assert np.allclose(orc.sgl(u, lam, 0.0, c, d), orc.grp_lasso(u, c * lam, d), atol=1e-14)
        assert np.allclose(orc.sgl(u, lam, 1.0, c, d), [orc.soft(x, lam, d) for x in u], atol=1e-14)


def test_sgl_lambda_max_is_smallest_null_fixed_point():
    rng = np.random.default_rng(34)
    p, ng = 12, 4
    group = np.repeat(np.arange(ng), 3)
    c = rng.normal(0, 1, p)
    w = rng.uniform(0.5, 1.5, p)
    for tau in (0.0, 0.3, 0.8, 1.0):
        lm = orc.lambda_max("sgl", c, w, group, ng, alpha=tau)
        G = np.eye(p)
        B0, _, _ = orc.oem_path(G, c, 1.0, "sgl", [lm], alpha=tau, w=w, group=group, ngroups=ng, maxit=1)
        B1, _, _ = orc.oem_path(G, c, 1.0, "sgl", [lm * (1 - 1e-3)], alpha=tau, w=w, group=group, ngroups=ng, maxit=1)
        assert not B0.any() and B1.any()
