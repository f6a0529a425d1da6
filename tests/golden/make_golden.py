"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every fixture stores the input *recipe* (NumPy PCG64 seed, shape, dtype), a
sha256 of the resulting fp64 matrix bytes (so a generator drift is caught),
and the reference outputs.  Matrices are drawn as float32 and widened to
float64 before the reference sees them (the parity protocol of SURVEY.md
§7.1: only arithmetic differs between engines, never input rounding).
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import gpspca  # noqa: E402  (the reference)
from gpspca import block as ref_block  # noqa: E402
from gpspca.single_unit import _solve_component  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from recipes import digest, make_matrix, polar_input  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sparse(z):
    z = np.asarray(z, dtype=np.float64)
    if z.ndim == 1:
        z = z[:, None]
    out = []
    for j in range(z.shape[1]):
        idx = np.nonzero(z[:, j])[0]
        out.append({"idx": idx.tolist(), "val": z[idx, j].tolist()})
    return out


def su_case(name, recipe, penalty, gamma_rule, **cfg):
    A = make_matrix(recipe)
    norms = gpspca.column_norms(A)
    gmax = float(norms.max())
    gamma = {"0.1max": 0.1 * gmax, "0.1max_sq": (0.1 * gmax) ** 2}.get(gamma_rule, gamma_rule)
    config = gpspca.SolverConfig(penalty=penalty, gamma=gamma, **cfg)
    loadings, report = gpspca.solve_single_unit(A, config)
    z, hist, conv, x = _solve_component(gpspca.DataMatrix(A), float(gamma), config,
                                        gpspca.parallel.DEFAULT_PLAN)
    assert np.array_equal(z, loadings.values[:, 0])
    return {
        "name": name, "solver": "single_unit", "recipe": recipe, "sha": digest(A),
        "penalty": penalty, "gamma": float(gamma), "config": cfg,
        "iterations": report.iterations, "converged": report.converged,
        "history": report.objective_history, "nnz": report.nnz_per_component,
        "z": sparse(loadings.values), "x": None if x is None else np.asarray(x).tolist(),
    }


def multi_case(name, recipe, penalty, gamma_rule, m, **cfg):
    A = make_matrix(recipe)
    gmax = float(gpspca.column_norms(A).max())
    gamma = {"0.1max": 0.1 * gmax, "0.1max_sq": (0.1 * gmax) ** 2}.get(gamma_rule, gamma_rule)
    config = gpspca.SolverConfig(penalty=penalty, gamma=gamma, m=m, **cfg)
    loadings, report = gpspca.solve_multi_sequential(A, config)
    return {
        "name": name, "solver": "multi_sequential", "recipe": recipe, "sha": digest(A),
        "penalty": penalty, "gamma": float(gamma), "m": m, "config": cfg,
        "iterations": report.iterations, "converged": report.converged,
        "histories": report.component_histories, "nnz": report.nnz_per_component,
        "z": sparse(loadings.values),
    }


def block_case(name, recipe, penalty, gamma_rule, m, mu=1.0, **cfg):
    A = make_matrix(recipe)
    gmax = float(gpspca.column_norms(A).max())
    gamma = {"0.1max": 0.1 * gmax, "0.1max_sq": (0.1 * gmax) ** 2, "0.02max": 0.02 * gmax,
             "0.02max_sq": (0.02 * gmax) ** 2}.get(gamma_rule, gamma_rule)
    mu_list = np.broadcast_to(np.asarray(mu, dtype=np.float64), (m,)).tolist()
    config = gpspca.SolverConfig(penalty=penalty, mode="block", gamma=gamma, m=m,
                                 mu=mu_list, **cfg)
    out = {
        "name": name, "solver": "block", "recipe": recipe, "sha": digest(A),
        "penalty": penalty, "gamma": float(gamma), "m": m, "mu": mu_list, "config": cfg,
    }
    try:
        loadings, report = gpspca.solve_block(A, config)
    except ref_block.RankDeficiencyError as err:
        out.update({"rank_error": {"rank": err.rank, "required": err.required,
                                   "iteration": err.iteration, "history": err.history}})
        return out
    out.update({
        "iterations": report.iterations, "converged": report.converged,
        "history": report.objective_history, "nnz": report.nnz_per_component,
        "z": sparse(loadings.values),
    })
    return out


def kernel_case():
    """Known-answer vectors for the kernel seam (parallel.py:85-142)."""
    recipe = {"kind": "gauss32", "seed": 7, "shape": [64, 1000]}
    A = make_matrix(recipe)
    rng = np.random.default_rng(8)
    x = rng.standard_normal(64)
    x /= np.linalg.norm(x)
    coef = rng.standard_normal(1000)
    c = gpspca.par_matvec_t(A, x)
    out = {"name": "kernels", "recipe": recipe, "sha": digest(A), "x": x.tolist(),
           "coef": coef.tolist(), "matvec_t": c.tolist(),
           "gram_apply": gpspca.par_gram_apply(A, coef).tolist()}
    for pen in ("l1", "l0"):
        gam = 0.5 if pen == "l1" else 0.25
        out[f"threshold_accumulate_{pen}"] = gpspca.par_threshold_accumulate(A, c, gam, pen).tolist()
        out[f"objective_{pen}"] = (gpspca.objective_sl1 if pen == "l1" else gpspca.objective_sl0)(A, x, gam)
        out[f"ascent_{pen}"] = (gpspca.ascent_direction_sl1 if pen == "l1"
                                else gpspca.ascent_direction_sl0)(A, x, gam).tolist()
        out[f"recover_{pen}"] = (gpspca.recover_pattern_sl1 if pen == "l1"
                                 else gpspca.recover_pattern_sl0)(A, x, gam).tolist()
    out["column_norms"] = gpspca.column_norms(A).tolist()
    G = rng.standard_normal((64, 6))
    out["polar_G"] = G.tolist()
    out["polar_X"] = gpspca.polar_projection(G).values.tolist()
    X = gpspca.polar_projection(rng.standard_normal((64, 3))).values
    out["block_X"] = X.tolist()
    out["block_gamma"] = [0.1, 0.2, 0.3]
    out["block_mu"] = [1.0, 0.8, 0.6]
    out["objective_bl1"] = gpspca.objective_bl1(A, X, out["block_gamma"], out["block_mu"])
    out["objective_bl0"] = gpspca.objective_bl0(A, X, out["block_gamma"], out["block_mu"])
    out["ascent_block_l1"] = gpspca.ascent_direction_block(
        A, X, out["block_gamma"], out["block_mu"], "l1").tolist()
    out["ascent_block_l0"] = gpspca.ascent_direction_block(
        A, X, out["block_gamma"], out["block_mu"], "l0").tolist()
    return out


def b64(M):
    import base64

    M = np.asfortranarray(M, dtype=np.float64)
    return {"shape": list(M.shape), "data": base64.b64encode(M.tobytes(order="F")).decode()}


def polar_case(name, recipe):
    """The reference polar_projection (block.py:135-149) on a conditioned G."""
    G = polar_input(recipe)
    # G and X are stored bit-exactly (base64 fp64, column-major): an
    # ill-conditioned G's polar factor moves with the last bits of G, so the
    # input must not depend on the LAPACK build that regenerates it
    out = {"name": name, "recipe": recipe, "sha": digest(G), "G": b64(G)}
    try:
        out["X"] = b64(ref_block.polar_projection(G).values)
    except ref_block.RankDeficiencyError as err:
        out["rank_error"] = {"rank": err.rank, "required": err.required}
    out["s"] = np.linalg.svd(G, compute_uv=False).tolist()
    return out


def hard_cases():
    """Round-2 fixtures: block solves at m = 32 / 64 (the C4 code paths:
    m_pad = 64 tensor-core refine / update, the CholeskyQR2 + Newton-Schulz
    polar step, CholeskyQR2 init at p m >= 4096), refine with deflation,
    near-collinear and duplicated max-norm columns at init."""
    lr64 = {"kind": "lowrank32", "seed": 31, "shape": [256, 4096], "rank": 64, "support": 32, "scale": 4.0}
    c1 = {"kind": "gauss32", "seed": 0, "shape": [500, 1000]}
    mu64 = np.linspace(1, 0.5, 64).tolist()
    return [
        block_case("lr64_bl0_m64_mu", lr64, "l0", "0.1max_sq", 64, mu=mu64),
        block_case("lr64_bl0_m64_mu_random", lr64, "l0", "0.1max_sq", 64, mu=mu64,
                   init="random_orthonormal", seed=5),
        block_case("lr64_bl0_m64_mu_random_g02", lr64, "l0", "0.02max_sq", 64, mu=mu64,
                   init="random_orthonormal", seed=5, max_iter=80),
        block_case("lr64_bl1_m32", lr64, "l1", "0.1max", 32),
        block_case("lr64_bl1_m32_random", lr64, "l1", "0.1max", 32, init="random_orthonormal", seed=6),
        block_case("lr64_bl1_m32_random_g02", lr64, "l1", "0.02max", 32, init="random_orthonormal", seed=6,
                   max_iter=80),
        block_case("c1_bl1_m64", c1, "l1", "0.1max", 64, max_iter=60),
        multi_case("c1_multi_sl1_m3_refine", c1, "l1", "0.1max", 3, refine=True),
        multi_case("c1_multi_sl0_m3_refine", c1, "l0", "0.1max_sq", 3, refine=True),
        block_case("nearcol_bl1_m2", {"kind": "nearcol", "seed": 41, "shape": [50, 300], "rel": 1e-9}, "l1",
                   "0.1max", 2),
        block_case("nearcol_bl1_m3", {"kind": "nearcol", "seed": 42, "shape": [50, 300], "rel": 1e-12}, "l1",
                   "0.1max", 3),
    ]


def init_error(case_fn, *args, **kw):
    try:
        return case_fn(*args, **kw)
    except ValueError as err:
        name, recipe = args[0], args[1]
        A = make_matrix(recipe)
        return {"name": name, "solver": "block", "recipe": recipe, "sha": digest(A), "penalty": args[2],
                "gamma": 0.1 * float(gpspca.column_norms(A).max()), "m": args[4], "mu": [1.0] * args[4],
                "config": {}, "init_error": str(err)}


def polar_cases():
    cases = []
    for m in (10, 64):
        for kappa in (10.0, 1e3, 1e5, 1e7):
            cases.append(polar_case(f"polar_m{m}_k{kappa:g}", {"seed": int(m + np.log10(kappa)),
                                                                "p": 512 if m == 10 else 128, "m": m,
                                                                "kappa": kappa}))
    cases.append(polar_case("polar_rank_keep", {"seed": 90, "p": 4096, "m": 2, "s": [89.9, 4.5e-10]}))
    cases.append(polar_case("polar_rank_drop", {"seed": 91, "p": 4096, "m": 2, "s": [89.9, 5e-11]}))
    cases.append(polar_case("polar_rank_zero", {"seed": 92, "p": 300, "m": 10,
                                                "s": [1.0] * 9 + [0.0]}))
    return cases


def main_hard():
    cases = hard_cases()
    cases.append(init_error(block_case, "dupcol_bl1_m2", {"kind": "nearcol", "seed": 43, "shape": [50, 300],
                                                          "rel": 0.0}, "l1", "0.1max", 2))
    with open(os.path.join(HERE, "solves_hard.json"), "w") as fh:
        json.dump({"reference": "gpspca 0.1.0 @ /root/reference/pkg", "numpy": np.__version__,
                   "cases": cases}, fh)
    with open(os.path.join(HERE, "polar.json"), "w") as fh:
        json.dump({"reference": "gpspca 0.1.0 @ /root/reference/pkg", "cases": polar_cases()}, fh)
    for c in cases:
        print(c["name"], c.get("iterations"), c.get("nnz"), "rank_error" in c, c.get("init_error"))


def main():
    c1 = {"kind": "gauss32", "seed": 0, "shape": [500, 1000]}
    cases = [
        su_case("c1_sl1", c1, "l1", "0.1max"),
        su_case("c1_sl0", c1, "l0", "0.1max_sq"),
        su_case("c1_sl1_random", c1, "l1", "0.1max", init="random_orthonormal", seed=3),
        su_case("c1_sl1_restarts", c1, "l1", "0.1max", restarts=3),
        su_case("c1_sl1_gamma0", c1, "l1", 0.0, tol=1e-10),
        multi_case("c1_multi_sl1_m5", c1, "l1", "0.1max", 5),
        multi_case("c1_multi_sl0_m3", c1, "l0", "0.1max_sq", 3),
        block_case("c1_bl1_m10", c1, "l1", "0.1max", 10),
        block_case("c1_bl0_m10_mu", c1, "l0", "0.1max_sq", 10, mu=np.linspace(1, 0.5, 10).tolist()),
        block_case("c1_bl1_m5_random", c1, "l1", "0.1max", 5, init="random_orthonormal", seed=0),
        block_case("c1_bl1_m1", c1, "l1", "0.1max", 1),
        # ragged shapes (p, n not multiples of any tile)
        su_case("ragged_sl1", {"kind": "gauss32", "seed": 11, "shape": [37, 1001]}, "l1", "0.1max"),
        su_case("ragged_sl0", {"kind": "gauss32", "seed": 12, "shape": [129, 515]}, "l0", "0.1max_sq"),
        block_case("ragged_bl1_m3", {"kind": "gauss32", "seed": 13, "shape": [37, 1001]}, "l1", "0.1max", 3),
        block_case("ragged_bl0_m4", {"kind": "gauss32", "seed": 14, "shape": [129, 515]}, "l0", "0.1max_sq", 4,
                   mu=[1.0, 0.9, 0.8, 0.7]),
        # low-rank + planted sparse factors (the C2/C3 distribution, scaled down)
        su_case("lowrank_sl0", {"kind": "lowrank32", "seed": 21, "shape": [256, 4096], "rank": 5,
                                "support": 40, "scale": 4.0}, "l0", "0.1max_sq"),
        su_case("lowrank_sl1", {"kind": "lowrank32", "seed": 21, "shape": [256, 4096], "rank": 5,
                                "support": 40, "scale": 4.0}, "l1", "0.1max"),
        block_case("lowrank_bl1_m5", {"kind": "lowrank32", "seed": 22, "shape": [256, 4096], "rank": 5,
                                      "support": 40, "scale": 4.0}, "l1", "0.1max", 5),
        # edge cases
        su_case("zeros", {"kind": "zeros", "seed": 0, "shape": [3, 4]}, "l1", 0.0),
        su_case("activation_limit", {"kind": "gauss32", "seed": 17, "shape": [4, 6]}, "l1", 100.0),
        su_case("diag_l0", {"kind": "diag", "seed": 0, "shape": [2, 2], "diag": [3.0, 1.0]}, "l0", 0.1),
        su_case("single_column", {"kind": "gauss32", "seed": 18, "shape": [50, 1]}, "l1", 0.5),
        su_case("single_row", {"kind": "gauss32", "seed": 19, "shape": [1, 300]}, "l0", 0.3),
        block_case("rank_collapse", {"kind": "diag", "seed": 0, "shape": [2, 2], "diag": [3.0, 0.1]}, "l0", 0.5, 2,
                   init="random_orthonormal", seed=1, max_iter=500),
    ]
    with open(os.path.join(HERE, "solves.json"), "w") as fh:
        json.dump({"reference": "gpspca 0.1.0 @ /root/reference/pkg", "numpy": np.__version__,
                   "cases": cases}, fh)
    with open(os.path.join(HERE, "kernels.json"), "w") as fh:
        json.dump(kernel_case(), fh)
    for c in cases:
        print(c["name"], c.get("iterations"), c.get("nnz"), "rank_error" in c)


if __name__ == "__main__":
    if "--hard" in sys.argv:
        main_hard()
    else:
        main()
