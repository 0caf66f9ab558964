"""Generate golden parity vectors by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``irksolve`` from /root/reference/pkg/src (read-only; numba's
cache is redirected to /tmp), feeds it inputs built by this repo's seeded
generators, and stores the reference outputs as compressed ``.npz`` files
next to this script.  The inputs themselves are NOT stored for the large
cases: they are regenerated bit-identically from (config, seed) at test time
and checked against the stored SHA-256 of the input arrays.
"""

from __future__ import annotations

import hashlib
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import irksolve as ref  # noqa: E402
from irksolve.kernels import set_backend  # noqa: E402

from paper_1701_07181_b200 import workloads as W  # noqa: E402
from paper_1701_07181_b200.meshes import build_mesh  # noqa: E402
from tests.helpers import random_blocks, sha  # noqa: E402

set_backend("numba")


def ref_graph(table_or_adj, partition_of=None):
    adj = [list(map(int, r)) for r in table_or_adj]
    g = ref.ElementGraph(num_elements=len(adj), adjacency=adj, periodic=True)
    if partition_of is not None:
        g = ref.ElementGraph(num_elements=len(adj), adjacency=adj, periodic=True,
                             partition_of=np.asarray(partition_of))
    return g


def ref_matrix(graph, data):
    mat = ref.BlockSparseMatrix(graph, data.shape[1])
    assert mat.data.shape == data.shape
    mat.data[:] = data
    return mat


def sample_idx(n, k=3):
    idx = sorted(set(list(range(min(k, n))) + list(range(max(0, n - k), n))
                     + list(range(0, n, max(1, n // 6)))))
    return np.array(idx, dtype=np.int64)


def solve_case(name, table, J, M, rhs, scheme, kind, restart, rtol, dt, partitions=None,
               store_full=False, max_iters=500):
    """Run the reference's operator, preconditioner and GMRES on one input."""
    tab = ref.builtin_tableau(scheme)
    der = ref.derive(tab)
    s = tab.s
    part = None
    if partitions:
        part = ref.partition(ref_graph(table), partitions).partition_of
    g = ref_graph(table)
    Jm = ref_matrix(g, J)
    mass = ref.BlockDiagonalMatrix(M)
    op = ref.StageOperator(der, dt, mass, [Jm] * s)
    rng = np.random.default_rng(99)
    w = rng.standard_normal(op.total_dim)
    y_mv = op.matvec(w)
    spec = ref.PrecondSpec(kind=kind, partitions=partitions)
    from irksolve.stepper import _make_preconditioner
    fac = _make_preconditioner(op, spec, part, None)
    y_ap = fac.apply(w) if fac is not None else w.copy()
    x, st = ref.gmres(op.matvec, None if fac is None else fac.apply, rhs,
                      ref.GmresConfig(rel_tol=rtol, restart=restart, max_iters=max_iters))
    out = dict(w=w, matvec=y_mv, apply=y_ap, x=x, iterations=st.iterations,
               operator_applies=st.operator_applies, converged=st.converged,
               residual_history=np.array(st.residual_history),
               final_true_residual=st.final_true_residual, dt=dt, a_inv=der.a_inv,
               shifts=der.shifts, input_sha=sha(J, M, rhs))
    # factor samples: dinv of sampled elements (all stages)
    T = len(table)
    idx = sample_idx(T)
    out["sample_elems"] = idx
    if kind in ("coupled", "coupled-literal"):
        out["dinv_sample"] = fac.dinv[:, idx]
        out["fcoupling_sample"] = fac.fcoupling[:, :, idx]
    elif fac is not None:
        out["dinv_sample"] = np.stack([f.dinv[idx] for f in fac.factors])
    if store_full:
        out.update(J=J, M=M, rhs=rhs)
        if kind in ("coupled", "coupled-literal"):
            out.update(fstage=fac.fstage, fcoupling=fac.fcoupling, dinv=fac.dinv)
        elif fac is not None:
            out.update(fdata=np.stack([f.fdata for f in fac.factors]),
                       dinv=np.stack([f.dinv for f in fac.factors]))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: T={T} s={s} kind={kind} iters={st.iterations} conv={st.converged} "
          f"true_res={st.final_true_residual:.3e}")


def kernel_cases():
    """Backend-protocol level cases (kernels/numba_backend.py) on small graphs."""
    from irksolve.kernels import numba_backend as nb
    out = {}
    # periodic line, like tests/test_backends.py
    g = ref.build_line_mesh(10, periodic=True)
    adj = g.adjacency
    data = random_blocks(adj, 3, seed=3)
    mat = ref_matrix(g, data)
    x = np.random.default_rng(2).standard_normal(mat.n)
    keep = np.ones(mat.nnz_blocks, dtype=bool)
    f, d, fail = nb.ilu0_factor(mat.indptr, mat.indices, mat.diag_pos, mat.data, keep, True)
    out["line_data"] = data
    out["line_x"] = x
    out["line_matvec"] = nb.bsr_matvec(mat.indptr, mat.indices, mat.data, x)
    out["line_f"], out["line_dinv"], out["line_fail"] = f, d, fail
    out["line_solve"] = nb.ilu0_solve(mat.indptr, mat.indices, mat.diag_pos, f, d, keep, x)
    # partitioned keep mask (P=4) on the same matrix
    gp = ref.partition(g, 4)
    keep4 = ref.partition_keep_mask(mat, gp.partition_of)
    f4, d4, _ = nb.ilu0_factor(mat.indptr, mat.indices, mat.diag_pos, mat.data, keep4, True)
    out["line_keep4"] = keep4
    out["line_f4"], out["line_dinv4"] = f4, d4
    out["line_solve4"] = nb.ilu0_solve(mat.indptr, mat.indices, mat.diag_pos, f4, d4, keep4, x)
    # general (non-simplified) path on the triangle graph
    tri_adj = [[1, 2], [0, 2], [0, 1]]
    tri = ref.ElementGraph(num_elements=3, adjacency=tri_adj)
    tdata = random_blocks(tri_adj, 2, seed=6, diag_boost=5.0)
    tmat = ref_matrix(tri, tdata)
    keep3 = np.ones(tmat.nnz_blocks, dtype=bool)
    tf, td, tfail = nb.ilu0_factor(tmat.indptr, tmat.indices, tmat.diag_pos, tmat.data, keep3,
                                   False)
    ty = np.random.default_rng(7).standard_normal(tmat.n)
    out["tri_data"], out["tri_f"], out["tri_dinv"], out["tri_fail"] = tdata, tf, td, tfail
    out["tri_y"] = ty
    out["tri_solve"] = nb.ilu0_solve(tmat.indptr, tmat.indices, tmat.diag_pos, tf, td, keep3, ty)
    # singular pivot at element 0 (tests/test_backends.py:76-84) and at element 2
    gl = ref.build_line_mesh(4)
    sdata = random_blocks(gl.adjacency, 2, seed=8)
    smat = ref_matrix(gl, sdata)
    smat.set_block(0, 0, np.zeros((2, 2)))
    out["sing_data0"] = smat.data.copy()
    out["sing_fail0"] = nb.ilu0_factor(smat.indptr, smat.indices, smat.diag_pos, smat.data,
                                       np.ones(smat.nnz_blocks, bool), True)[2]
    smat2 = ref_matrix(gl, sdata)
    # make the pivot of element 2 numerically singular after the Schur update:
    # B22 = L21 U12 + u v^T, so D2 = u v^T + O(eps) has cond ~ 1e16 > COND_LIMIT
    # on any summation order (a rank-0 D2 would hinge on exact cancellation)
    f_ok, d_ok, _ = nb.ilu0_factor(smat2.indptr, smat2.indices, smat2.diag_pos, smat2.data,
                                   np.ones(smat2.nnz_blocks, bool), True)
    k21 = smat2._pos(2, 1)
    k12 = smat2._pos(1, 2)
    smat2.set_block(2, 2, f_ok[k21] @ smat2.data[k12] + np.outer([1.0, 2.0], [0.5, -1.0]))
    out["sing_data2"] = smat2.data.copy()
    out["sing_fail2"] = nb.ilu0_factor(smat2.indptr, smat2.indices, smat2.diag_pos, smat2.data,
                                       np.ones(smat2.nnz_blocks, bool), True)[2]
    # coupled factor/solve on RADAU35 with distinct J_k (tests/test_backends.py:20-27)
    tab = ref.builtin_tableau("RADAU35")
    der = ref.derive(tab)
    T, m = 8, 3
    rng = np.random.default_rng(0)
    Mb = np.eye(m) + 0.05 * rng.standard_normal((T, m, m))
    gl8 = ref.build_line_mesh(T, periodic=True)
    jdata = [random_blocks(gl8.adjacency, m, seed=1 + k) for k in range(tab.s)]
    jacs = [ref_matrix(gl8, d_) for d_ in jdata]
    op = ref.StageOperator(der, 0.08, ref.BlockDiagonalMatrix(Mb), jacs)
    wv = np.random.default_rng(5).standard_normal(op.total_dim)
    out["cpl_J"] = np.stack(jdata)
    out["cpl_M"] = Mb
    out["cpl_w"] = wv
    out["cpl_matvec"] = op.matvec(wv)
    for lit in (False, True):
        cf = ref.stage_coupled_factorize(op, literal_update=lit)
        tag = "lit" if lit else "std"
        out[f"cpl_{tag}_fstage"] = cf.fstage
        out[f"cpl_{tag}_fcoupling"] = cf.fcoupling
        out[f"cpl_{tag}_dinv"] = cf.dinv
        out[f"cpl_{tag}_apply"] = cf.apply(wv)
    uf = ref.stage_uncoupled_factorize(op, der.shifts)
    out["unc_apply"] = uf.apply(wv)
    out["unc_dinv"] = np.stack([f.dinv for f in uf.factors])
    out["unc_fdata"] = np.stack([f.fdata for f in uf.factors])
    uf0 = ref.stage_uncoupled_factorize(op, None)
    out["unc0_apply"] = uf0.apply(wv)
    bj = ref.stage_uncoupled_factorize(op, der.shifts, partition_of=np.arange(T))
    out["bj_apply"] = bj.apply(wv)
    cp4 = ref.stage_coupled_factorize(op, partition_of=ref.partition(gl8, 4).partition_of)
    out["cpl4_apply"] = cp4.apply(wv)
    # GMRES on the coupled/uncoupled model operator (tests/test_precond.py:208-218)
    rhs = np.random.default_rng(9).standard_normal(op.total_dim)
    out["gm_rhs"] = rhs
    for tag, fac in (("cpl", ref.stage_coupled_factorize(op)), ("unc", uf)):
        xg, st = ref.gmres(op.matvec, fac.apply, rhs, ref.GmresConfig(rel_tol=1e-8))
        out[f"gm_{tag}_x"] = xg
        out[f"gm_{tag}_iters"] = st.iterations
        out[f"gm_{tag}_hist"] = np.array(st.residual_history)
        xr, st = ref.gmres(op.matvec, fac.apply, rhs, ref.GmresConfig(rel_tol=1e-10, restart=3))
        out[f"gm_{tag}_rst_x"] = xr
        out[f"gm_{tag}_rst_iters"] = st.iterations
    # tableau KATs
    for name in ("RADAU23", "RADAU35", "DIRK33"):
        d_ = ref.derive(ref.builtin_tableau(name))
        out[f"tab_{name}_a_inv"] = d_.a_inv
        out[f"tab_{name}_shifts"] = d_.shifts
    np.savez_compressed(os.path.join(HERE, "kernels_small.npz"), **out)
    print("kernels_small written")


def workload_case(name, cfg, kind=None, partitions=None, store_full=False, max_iters=500):
    wl = W.make_workload(cfg)
    solve_case(name, wl.table, wl.J, wl.M, wl.rhs, cfg.scheme, kind or cfg.precond,
               cfg.restart, cfg.rtol, wl.dt, partitions=partitions, store_full=store_full,
               max_iters=max_iters)


def dirk_case():
    """DIRK33 implicit stage (stepper.py:268-274) on a small 2D mesh."""
    cfg = W.CONFIGS[1].scaled(N=6, nb=8)
    wl = W.make_workload(cfg)
    g = ref_graph(wl.table)
    Jm = ref_matrix(g, wl.J)
    mass = ref.BlockDiagonalMatrix(wl.M)
    tab = ref.builtin_tableau("DIRK33")
    aii = tab.A[0, 0]
    mat = ref.build_stage_matrix(1.0, mass, Jm, wl.dt * aii)
    fac = ref.ilu0_factorize(mat)
    n = mat.n
    rhs = wl.rhs[:n]
    x, st = ref.gmres(mat.matvec, fac.apply, rhs, ref.GmresConfig(rel_tol=1e-8, restart=40))
    w = np.random.default_rng(3).standard_normal(n)
    np.savez_compressed(os.path.join(HERE, "dirk_small.npz"), x=x, iterations=st.iterations,
                        matvec=mat.matvec(w), apply=fac.apply(w), w=w, dt=wl.dt, aii=aii,
                        input_sha=sha(wl.J, wl.M, wl.rhs))
    print(f"dirk_small: iters={st.iterations}")


def stepper_cases():
    """Newton time steps (stepper.py:127-181, 229-287) on the linear problem
    M du/dt = J u (BASELINE config 4's "rhs = J.u"), config-1 mesh shape reduced
    (N=6, nb=8): RADAU23 coupled, RADAU35 shifted uncoupled, DIRK33; two steps each,
    with the reference's OpCounter."""
    from irksolve.problems import SemidiscreteProblem
    from irksolve.stepper import NewtonConfig, PrecondSpec, dirk_step, irk_step_transformed

    out = {}
    for dtn in (10.0, 100.0):
        cfg = W.CONFIGS[1].scaled(N=6, nb=8, dt_norm=dtn)
        wl = W.make_workload(cfg)
        g = ref_graph(wl.table)
        Jm = ref_matrix(g, wl.J)
        mass = ref.BlockDiagonalMatrix(wl.M)
        u0 = np.random.default_rng(11).standard_normal(Jm.n)

        class LinearJ(SemidiscreteProblem):
            name = "linear-J"

            def __init__(self):
                self.graph = g
                self.m = wl.J.shape[1]

            def mass(self):
                return mass

            def rhs(self, t, u):
                return Jm.matvec(u)

            def jacobian(self, t, u):
                return Jm

        prob = LinearJ()
        gcfg = ref.GmresConfig(rel_tol=1e-8, restart=40)
        tag = f"dt{int(dtn)}"
        out[f"{tag}_dt"] = wl.dt
        out[f"{tag}_u0"] = u0
        out[f"{tag}_sha"] = sha(wl.J, wl.M)
        for name, scheme, kind in (("r23c", "RADAU23", "coupled"), ("r35u", "RADAU35", "uncoupled"),
                                   ("dirk", "DIRK33", None)):
            tab = ref.builtin_tableau(scheme)
            u = u0.copy()
            ctr = ref.OpCounter()
            for step in range(2):
                if kind is None:
                    res = dirk_step(prob, tab, u, step * wl.dt, wl.dt, NewtonConfig(), gcfg, ctr)
                else:
                    res = irk_step_transformed(prob, tab, u, step * wl.dt, wl.dt, PrecondSpec(kind=kind),
                                               NewtonConfig(), gcfg, ctr)
                u = res.u_next
                out[f"{tag}_{name}_u{step + 1}"] = u
                out[f"{tag}_{name}_newton{step + 1}"] = res.newton_iterations
                out[f"{tag}_{name}_gmres{step + 1}"] = np.array([st.iterations for st in res.gmres_stats])
            out[f"{tag}_{name}_counter"] = np.array([ctr.block_multiplies, ctr.block_solves,
                                                     ctr.block_factorizations, ctr.mass_multiplies,
                                                     ctr.jacobian_multiplies])
            print(f"stepper {tag} {name}: newton {out[f'{tag}_{name}_newton1']} "
                  f"gmres {out[f'{tag}_{name}_gmres1']}")
    np.savez_compressed(os.path.join(HERE, "stepper_small.npz"), **out)


def text_format_case():
    """Reference dump_matrix (blocks.py:193-201) on a small matrix: the exact text."""
    from irksolve.blocks import dump_matrix
    g = ref.build_line_mesh(6, periodic=True)
    mat = ref_matrix(g, random_blocks(g.adjacency, 3, seed=21))
    mat.data[0, 0, 0] = 1e-300
    mat.data[1, 1, 1] = -0.1
    mat.data[2, 2, 2] = 12345678901234.5
    dump_matrix(mat, os.path.join(HERE, "matrix_line6.txt"))
    print("matrix_line6.txt written")


def tableau_partition_cases():
    """Round-2 KATs: every builtin tableau (A, b, c, order, derive) including the
    generated RADAU47/RADAU59 and ESDIRK65 (tableaux.py:140-275), the s-stage
    generator for s = 1..9, and the reference partition map for T % P != 0
    (meshing.py:81-90)."""
    out = {}
    for name in ref.tableaux.BUILTIN_NAMES:
        tab = ref.builtin_tableau(name)
        d_ = ref.derive(tab)
        for k, v in (("A", tab.A), ("b", tab.b), ("c", tab.c), ("a_inv", d_.a_inv),
                     ("bT_a_inv", d_.bT_a_inv), ("shifts", d_.shifts)):
            out[f"{name}_{k}"] = np.asarray(v)
        out[f"{name}_order"] = tab.order
        out[f"{name}_kind"] = tab.kind.value
    for s in range(1, 10):
        tab = ref.tableaux.generate_radau_iia(s)
        out[f"gen{s}_A"], out[f"gen{s}_c"] = tab.A, tab.c
    for T, P in ((50, 4), (7, 3), (10, 10), (3072, 8), (101, 8), (12, 5)):
        g = ref.build_line_mesh(T, periodic=True)
        out[f"part_{T}_{P}"] = ref.partition(g, P).partition_of
    np.savez_compressed(os.path.join(HERE, "tableaux_r2.npz"), **out)
    print("tableaux_r2 written")


def stepper_cases_r2():
    """Newton steps with the s = 4 / 5 Radau IIA tableaux (generated) and the
    ESDIRK65 explicit first stage (stepper.py:253-259: one mass solve), on the
    same linear problem and shapes as stepper_cases."""
    from irksolve.problems import SemidiscreteProblem
    from irksolve.stepper import NewtonConfig, PrecondSpec, dirk_step, irk_step_transformed

    out = {}
    cfg = W.CONFIGS[1].scaled(N=6, nb=8, dt_norm=10.0)
    wl = W.make_workload(cfg)
    g = ref_graph(wl.table)
    Jm = ref_matrix(g, wl.J)
    mass = ref.BlockDiagonalMatrix(wl.M)
    u0 = np.random.default_rng(11).standard_normal(Jm.n)

    class LinearJ(SemidiscreteProblem):
        name = "linear-J"

        def __init__(self):
            self.graph = g
            self.m = wl.J.shape[1]

        def mass(self):
            return mass

        def rhs(self, t, u):
            return Jm.matvec(u)

        def jacobian(self, t, u):
            return Jm

    prob = LinearJ()
    gcfg = ref.GmresConfig(rel_tol=1e-8, restart=40)
    out["dt"], out["u0"], out["sha"] = wl.dt, u0, sha(wl.J, wl.M)
    for name, scheme, kind in (("r47u", "RADAU47", "uncoupled"), ("r47c", "RADAU47", "coupled"),
                               ("r59u", "RADAU59", "uncoupled"), ("r59c", "RADAU59", "coupled"),
                               ("esdirk", "ESDIRK65", None)):
        tab = ref.builtin_tableau(scheme)
        u = u0.copy()
        ctr = ref.OpCounter()
        for step in range(2):
            if kind is None:
                res = dirk_step(prob, tab, u, step * wl.dt, wl.dt, NewtonConfig(), gcfg, ctr)
            else:
                res = irk_step_transformed(prob, tab, u, step * wl.dt, wl.dt, PrecondSpec(kind=kind),
                                           NewtonConfig(), gcfg, ctr)
            u = res.u_next
            out[f"{name}_u{step + 1}"] = u
            out[f"{name}_newton{step + 1}"] = res.newton_iterations
            out[f"{name}_gmres{step + 1}"] = np.array([st.iterations for st in res.gmres_stats])
        out[f"{name}_counter"] = np.array([ctr.block_multiplies, ctr.block_solves,
                                           ctr.block_factorizations, ctr.mass_multiplies,
                                           ctr.jacobian_multiplies])
        print(f"stepper_r2 {name}: newton {out[f'{name}_newton1']} gmres {out[f'{name}_gmres1']}")
    np.savez_compressed(os.path.join(HERE, "stepper_r2.npz"), **out)


def cfg2_nb50_cases():
    """Config-2 shape at its real block size (nb=50, s=3, shifted uncoupled,
    GMRES(40), dt||J||2=100) on the 8^3-cube Kuhn mesh (T=3072), solved by the
    reference at P = 1, 2, 4, 8 (partition(graph, P), precond.py:26-45), natural
    numbering, plus the slab-colour numbering at P = 8.  Vectors are 460,800
    long, so only strided samples (every 61st entry) and full norms are stored;
    the GPU tests compare full vectors against the oracle and these samples
    against the reference."""
    cfg = W.CONFIGS[2].scaled(N=8)
    cases = [("natural", P) for P in (1, 2, 4, 8)] + [("color", 8)]
    for ordering, P in cases:
        c = cfg.scaled(ordering=ordering, extra={"parts": P} if ordering == "color" else {})
        wl = W.make_workload(c)
        tab = ref.builtin_tableau(c.scheme)
        der = ref.derive(tab)
        s = tab.s
        g = ref_graph(wl.table)
        part = ref.partition(g, P).partition_of if P > 1 else None
        Jm = ref_matrix(g, wl.J)
        mass = ref.BlockDiagonalMatrix(wl.M)
        op = ref.StageOperator(der, wl.dt, mass, [Jm] * s)
        w = np.random.default_rng(99).standard_normal(op.total_dim)
        from irksolve.stepper import _make_preconditioner
        fac = _make_preconditioner(op, ref.PrecondSpec(kind=c.precond, partitions=P if P > 1 else None),
                                   part, None)
        y_mv, y_ap = op.matvec(w), fac.apply(w)
        x, st = ref.gmres(op.matvec, fac.apply, wl.rhs,
                          ref.GmresConfig(rel_tol=c.rtol, restart=c.restart))
        idx = np.arange(0, op.total_dim, 61)
        out = dict(idx=idx, matvec=y_mv[idx], apply=y_ap[idx], x=x[idx],
                   matvec_norm=np.linalg.norm(y_mv), apply_norm=np.linalg.norm(y_ap),
                   x_norm=np.linalg.norm(x), iterations=st.iterations, converged=st.converged,
                   residual_history=np.array(st.residual_history),
                   final_true_residual=st.final_true_residual, dt=wl.dt, jnorm=wl.jnorm,
                   input_sha=sha(wl.J, wl.M, wl.rhs), w_sha=sha(w))
        name = f"cfg2_n8_nb50_{ordering}_p{P}"
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(f"{name}: iters={st.iterations} conv={st.converged} true_res={st.final_true_residual:.3e}",
              flush=True)


def main():
    if "--r2" in sys.argv:
        tableau_partition_cases()
        stepper_cases_r2()
        if "--no-cfg2" not in sys.argv:
            cfg2_nb50_cases()
        return
    if "--text" in sys.argv:
        text_format_case()
        return
    if "--stepper" in sys.argv:
        stepper_cases()
        return
    kernel_cases()
    stepper_cases()
    text_format_case()
    dirk_case()
    # config 0 exactly (2D tri 16x16, nb=24, RADAU23, coupled GMRES(30))
    workload_case("cfg0", W.CONFIGS[0])
    # config-1 shape on a reduced mesh (8x8 quads), shifted uncoupled GMRES(40)
    workload_case("cfg1_n8", W.CONFIGS[1].scaled(N=8), store_full=False)
    # same, colour-major numbering (a different ILU(0), its own oracle run)
    workload_case("cfg1_n8_color", W.CONFIGS[1].scaled(N=8, ordering="color"))
    # coupled preconditioner on the config-1 shape (config 4 comparator)
    workload_case("cfg1_n6_coupled", W.CONFIGS[1].scaled(N=6, scheme="RADAU23"), kind="coupled")
    # 3D Kuhn tets, config-2 shape reduced (4^3 cubes, nb=10), P=1 and P=4
    c2 = W.CONFIGS[2].scaled(N=4, nb=10)
    workload_case("cfg2_n4", c2)
    workload_case("cfg2_n3_full", c2.scaled(N=3, nb=6), store_full=True)
    workload_case("cfg2_n4_p4", c2, partitions=4)
    workload_case("cfg2_n4_color", c2.scaled(ordering="color"))
    # variance reading (stress): pinned max_iters so both sides stop together
    workload_case("cfg1_n8_var", W.CONFIGS[1].scaled(N=8, jstd="sqrtnb"), max_iters=60)


if __name__ == "__main__":
    main()
