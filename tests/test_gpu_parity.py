"""GPU parity: the CUDA path through the C ABI vs the oracle, element by element on the
same seeded inputs (BASELINE.json north_star tolerances: pattern and maps bit-exact,
≤ 1e-12 relative Frobenius per element matrix, ≤ 1e-11 on K's values; tables
≤ 1e-13, coefficients ≤ 1e-12; sensitivity ≤ 1e-11 relative 2-norm — DESIGN.md §5)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import parity_tools as PT

TOL_TABLE = 1e-13
TOL_COEF = 1e-12   # κ(V1)^d rounding amplification: 6.48^3 ≈ 272 at q=3
TOL_ELEM = 1e-12
TOL_K = 1e-11
TOL_SENS = 1e-11

_gpu = {}


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def gpu_case(c, **kw):
    """Build the Assembler and run assemble (+ local values) for config c (cached)."""
    key = (c, tuple(sorted(kw.items())))
    if key in _gpu:
        return _gpu[key]
    from paper_2107_09568_b200 import Assembler
    from synth import make_config
    prob = make_config(c, **kw)
    A = Assembler(prob)
    s = A.sizes
    dev = torch.device("cuda:0")
    ctrl = torch.tensor(prob.macro.ctrl, dtype=torch.float64, device=dev)
    young = torch.tensor(prob.young, dtype=torch.float64, device=dev)
    vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
    keep_local = s.n_local_rows * s.n_tiles * prob.d ** 2 < 3e9
    local = torch.empty(s.n_local_rows * s.n_tiles * prob.d ** 2, dtype=torch.float64, device=dev) if keep_local else None
    A.assemble(ctrl, young, prob.nu, vals, local)
    torch.cuda.synchronize()
    out = dict(prob=prob, A=A, ctrl=ctrl, young=young, vals=vals, local=local)
    _gpu[key] = out
    return out


def local_np(g, tiles):
    """GPU element matrices of the given tiles: (len, n_rows, d, d)."""
    prob, s = g["prob"], g["A"].sizes
    d = prob.d
    L = g["local"].view(s.n_local_rows, s.n_tiles, d, d)
    return L[:, torch.as_tensor(tiles, device=L.device)].permute(1, 0, 2, 3).cpu().numpy()


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("c", [1, 2, 3])
def test_tables_parity(c, oracle_problem):
    """All patch tables (cfg4/cfg5: tests/test_gpu_fullsize.py)."""
    g = gpu_case(c)
    ob = oracle_problem(c)
    Tg = g["A"].tables()
    assert np.array_equal(g["A"].pairs(), np.concatenate(ob["tabs"].pairs))
    off = 0
    for Tp, _ in ob["tabs"].per_patch:
        assert rel(Tg[off:off + len(Tp)], Tp) < TOL_TABLE
        off += len(Tp)


@pytest.mark.parametrize("c", [1, 2, 3, 4])
def test_interpolation_parity(c):
    from oracle import macro as M
    g = gpu_case(c)
    prob, A = g["prob"], g["A"]
    s = A.sizes
    d = prob.d
    coef = torch.zeros(s.n_tiles * d * d * s.k_stride, dtype=torch.float64, device="cuda")
    A.interpolate(g["ctrl"], g["young"], prob.nu, coef)
    cg = coef.view(s.n_tiles, d * d, s.k_stride)[:, :, :s.n_k].cpu().numpy()
    tiles = range(prob.n_tiles)
    for t in tiles:
        ref = M.tile_coefficients(prob, prob.macro.ctrl, int(t))            # [C, i, j, a, b]
        refm = np.transpose(ref, (3, 4, 1, 2, 0)).reshape(d * d, -1)          # [(a,b)][(i,j,C)]
        assert rel(cg[t], refm) < TOL_COEF, t
    # padding columns stay zero
    assert torch.count_nonzero(coef.view(s.n_tiles, d * d, s.k_stride)[:, :, s.n_k:]) == 0


@pytest.mark.parametrize("c", [1, 2, 3])
def test_element_matrix_parity(c, oracle_problem):
    """Every tile (cfg4/cfg5: tests/test_gpu_fullsize.py)."""
    from oracle import assemble as As
    g = gpu_case(c)
    prob = g["prob"]
    tabs = oracle_problem(c)["tabs"]
    tiles = list(range(prob.n_tiles))
    ref = As.local_lookup(prob, tabs, prob.macro.ctrl, tiles)
    got = local_np(g, tiles)
    for n, t in enumerate(tiles):
        assert rel(got[n], ref[n]) < TOL_ELEM, (t, rel(got[n], ref[n]))


@pytest.mark.parametrize("c", [1, 2, 3])
def test_pattern_bit_exact(c, oracle_problem):
    g = gpu_case(c)
    ob = oracle_problem(c)
    s = g["A"].sizes
    rp = torch.empty(s.n_dof + 1, dtype=torch.int64, device="cuda")
    ci = torch.empty(s.nnz, dtype=torch.int32, device="cuda")
    g["A"].pattern(rp, ci)
    assert np.array_equal(rp.cpu().numpy(), ob["pattern"].row_ptr)
    PT.check_col_idx(ci, ob["pattern"], g["prob"].d)                   # every entry
    bm = g["A"].block_map(0, prob_tiles(g))                            # every tile
    assert np.array_equal(bm, ob["pattern"].block_map())
    nl = sum(t.n_ctrl for t in g["prob"].tile)
    assert np.array_equal(g["A"].node_map_for(nl), ob["dm"].node)


def prob_tiles(g):
    return g["prob"].n_tiles


@pytest.mark.parametrize("c", [1, 2, 3])
def test_csr_values_parity(c, oracle_problem):
    from oracle import assemble as As
    g = gpu_case(c)
    ob = oracle_problem(c)
    vals_ref, _ = As.assemble_lookup(ob["prob"], ob["tabs"], ob["pattern"])
    got = g["vals"].cpu().numpy()
    assert rel(got, vals_ref) < TOL_K


@pytest.mark.parametrize("c", [1, 2, 3])
def test_K_bitwise_symmetric_and_deterministic(c):
    g = gpu_case(c)
    A, prob = g["A"], g["prob"]
    s = A.sizes
    rp = torch.empty(s.n_dof + 1, dtype=torch.int64, device="cuda")
    ci = torch.empty(s.nnz, dtype=torch.int32, device="cuda")
    A.pattern(rp, ci)
    K = torch.sparse_csr_tensor(rp, ci.to(torch.int64), g["vals"], size=(s.n_dof, s.n_dof))
    Kt = K.to_sparse_coo().t().coalesce()
    Kc = K.to_sparse_coo().coalesce()
    assert torch.equal(Kt.indices(), Kc.indices()) and torch.equal(Kt.values(), Kc.values())
    vals2 = torch.empty_like(g["vals"])
    A.assemble(g["ctrl"], g["young"], prob.nu, vals2)
    assert torch.equal(vals2, g["vals"])
    # rigid translations in the kernel (any F)
    for a in range(prob.d):
        tr = torch.zeros(s.n_dof, dtype=torch.float64, device="cuda")
        tr[a::prob.d] = 1.0
        r = torch.mv(K, tr).abs().max().item()
        assert r < 1e-11 * g["vals"].abs().max().item()


def test_host_pointers_match_device_pointers():
    """The [any]-pointer contract: host numpy buffers give the same bits (e2e path)."""
    g = gpu_case(2)
    prob, A = g["prob"], g["A"]
    vals_h = np.empty(A.sizes.nnz)
    A.assemble(np.ascontiguousarray(prob.macro.ctrl), np.ascontiguousarray(prob.young), prob.nu, vals_h)
    assert np.array_equal(vals_h, g["vals"].cpu().numpy())


def test_concurrent_calls_on_one_handle():
    """include/iga.h Concurrency: calls on one handle from several host threads, each on its
    own stream, are serialised by the handle's lock — every result equals its serial value
    bit for bit (without the lock they would race on the coefficient and side-slot workspace)."""
    import threading
    g = gpu_case(3)
    prob, A = g["prob"], g["A"]
    dev = g["vals"].device
    young2 = 2.0 * g["young"]
    u = torch.randn(A.sizes.n_dof, dtype=torch.float64, device=dev, generator=torch.Generator(device=dev).manual_seed(5))
    grad_ref = torch.empty(A.sizes.n_macro_cp * prob.d, dtype=torch.float64, device=dev)
    A.sensitivity(g["ctrl"], g["young"], prob.nu, u, u, grad_ref)
    vals2_ref = torch.empty_like(g["vals"])
    A.assemble(g["ctrl"], young2, prob.nu, vals2_ref)
    torch.cuda.synchronize()
    errs = []

    def worker(kind, reps=4):
        st = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(st):
            for _ in range(reps):
                if kind == 0:
                    v = torch.empty_like(g["vals"])
                    A.assemble(g["ctrl"], g["young"], prob.nu, v, stream=st)
                    ok = torch.equal(v, g["vals"])
                elif kind == 1:
                    v = torch.empty_like(g["vals"])
                    A.assemble(g["ctrl"], young2, prob.nu, v, stream=st)
                    ok = torch.equal(v, vals2_ref)
                else:
                    gr = torch.empty_like(grad_ref)
                    A.sensitivity(g["ctrl"], g["young"], prob.nu, u, u, gr, stream=st)
                    ok = torch.equal(gr, grad_ref)
                if not ok:
                    errs.append(kind)

    th = [threading.Thread(target=worker, args=(k,)) for k in (0, 1, 2, 0)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, f"results differ from the serial ones in workers {errs}"


def test_young_scaling_and_homogeneity_gpu():
    g = gpu_case(2)
    prob, A = g["prob"], g["A"]
    v2 = torch.empty_like(g["vals"])
    A.assemble(2.0 * g["ctrl"], g["young"], prob.nu, v2)          # K(2P) = 2 K(P) in 3D, bitwise
    assert torch.equal(v2, 2.0 * g["vals"])
    A.assemble(g["ctrl"], 3.0 * g["young"], prob.nu, v2)          # K(3E) = 3 K(E) (λ, μ ∝ E)
    assert (torch.linalg.norm(v2 - 3.0 * g["vals"]) / torch.linalg.norm(3.0 * g["vals"])).item() < 1e-14


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("c,kw", [(1, {}), (2, dict(n_el=(2, 1, 1))), (2, {})])
def test_sensitivity_parity(c, kw, oracle_problem):
    from oracle import sensitivity as S
    from synth import draw_uv_seeded
    ob = oracle_problem(c, **kw)
    g = gpu_case(c, **kw)
    prob, A = g["prob"], g["A"]
    u, v = draw_uv_seeded(c, ob["dm"].n_dof)
    ref = S.sensitivity(ob["prob"], ob["tabs"], ob["pattern"], u, v)
    grad = torch.empty(A.sizes.n_macro_cp * prob.d, dtype=torch.float64, device="cuda")
    A.sensitivity(g["ctrl"], g["young"], prob.nu, torch.tensor(u, device="cuda"), torch.tensor(v, device="cuda"), grad)
    got = grad.cpu().numpy().reshape(-1, prob.d)
    assert rel(got, ref) < TOL_SENS, rel(got, ref)


def test_sensitivity_cfg3_complete(oracle_problem):
    """The complete cfg3 gradient (3000 entries) against the oracle's complex step."""
    from synth import draw_uv_seeded
    ob = oracle_problem(3)
    g = gpu_case(3)
    prob, A = g["prob"], g["A"]
    u, v = draw_uv_seeded(3, A.sizes.n_dof)
    grad = torch.empty(A.sizes.n_macro_cp * 3, dtype=torch.float64, device="cuda")
    A.sensitivity(g["ctrl"], g["young"], prob.nu, torch.tensor(u, device="cuda"), torch.tensor(v, device="cuda"), grad)
    got = grad.cpu().numpy().reshape(-1, 3)
    assert np.abs(got.sum(0)).max() < 1e-10 * np.abs(got).max()          # translation invariance
    parts = PT.run(PT.w_sensitivity, PT.tile_chunks(prob.n_tiles, 8), prob=ob["prob"], tabs=ob["tabs"],
                   pattern=ob["pattern"], u=u, v=v)
    ref = np.sum(parts, axis=0)
    assert rel(got, ref) < TOL_SENS, rel(got, ref)


# ---------------------------------------------------------------------------
def test_degenerate_macro_raises():
    from paper_2107_09568_b200 import IgaError
    g = gpu_case(1)
    prob, A = g["prob"], g["A"]
    bad = prob.macro.ctrl.copy()
    bad[7, 0] += 3.0                     # drag an interior point across two elements: folds F
    vals = torch.empty(A.sizes.nnz, dtype=torch.float64, device="cuda")
    with pytest.raises(IgaError, match="EDEGENERATE"):
        A.assemble(torch.tensor(bad, device="cuda"), g["young"], prob.nu, vals)
    # the handle stays usable afterwards
    A.assemble(g["ctrl"], g["young"], prob.nu, vals)
    assert torch.equal(vals, g["vals"])


def test_invalid_arguments_raise():
    from paper_2107_09568_b200 import Assembler, IgaError
    from synth import make_config
    g = gpu_case(1)
    prob, A = g["prob"], g["A"]
    vals = torch.empty(A.sizes.nnz, dtype=torch.float64, device="cuda")
    with pytest.raises(IgaError, match="EINVAL"):
        A.assemble(g["ctrl"], g["young"], 0.5, vals)
    p2 = make_config(1)
    p2.tile[0].ctrl[6, 1] += 1e-3
    with pytest.raises(IgaError, match="ENONCONFORMING"):
        Assembler(p2)
    p3 = make_config(1)
    p3.tile[0].ctrl[14] = p3.tile[0].ctrl[15] + np.array([0.3, 0.0])   # folds the tile
    with pytest.raises(IgaError, match="EDEGENERATE|EINVAL"):
        Assembler(p3)


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("c,n", [(2, 2), (3, 3)])
def test_sharded_assembly_and_gradient(c, n):
    """One problem in n slabs (iga_shard): each shard's CSR rows are
    bit-identical to the whole problem's rows, and the shards' partial gradients sum to
    the whole gradient (the all-reduce of the multi-GPU step, done here on one GPU)."""
    from paper_2107_09568_b200 import Assembler
    from synth import draw_uv_seeded
    g = gpu_case(c)
    prob, A = g["prob"], g["A"]
    s = A.sizes
    rp = torch.empty(s.n_dof + 1, dtype=torch.int64, device="cuda")
    A.pattern(rp, None)
    rp = rp.cpu().numpy()
    u, v = draw_uv_seeded(c, s.n_dof)
    ut, vt = torch.tensor(u, device="cuda"), torch.tensor(v, device="cuda")
    gfull = torch.empty(s.n_macro_cp * prob.d, dtype=torch.float64, device="cuda")
    A.sensitivity(g["ctrl"], g["young"], prob.nu, ut, vt, gfull)
    gsum = torch.zeros_like(gfull)
    for k in range(n):
        B = Assembler(prob, shard=(n, k))
        z = B.sizes
        vals = torch.empty(z.nnz, dtype=torch.float64, device="cuda")
        B.assemble(g["ctrl"], g["young"], prob.nu, vals)
        a, b = rp[z.row_begin], rp[z.row_begin + z.n_rows]
        assert torch.equal(vals, g["vals"][a:b]), k
        gk = torch.empty_like(gfull)
        B.sensitivity(g["ctrl"], g["young"], prob.nu, ut, vt, gk)
        gsum += gk
    assert (torch.linalg.norm(gsum - gfull) / torch.linalg.norm(gfull)).item() < 1e-13


# ---------------------------------------------------------------------------
# matrix-free apply (NEXT N1, Eq. 74): y = K^π u without forming K

@pytest.mark.parametrize("c", [1, 2, 3])
def test_matrix_free_apply(c, oracle_problem):
    """iga_apply equals the oracle's assembled K times u (≤ 1e-11 rel.) and the GPU CSR
    product (≤ 1e-12 rel.); bitwise deterministic."""
    import scipy.sparse as sp
    from oracle import assemble as As
    from synth import draw_uv_seeded
    g = gpu_case(c)
    prob, A = g["prob"], g["A"]
    s = A.sizes
    u, _ = draw_uv_seeded(c, s.n_dof)
    ut = torch.tensor(u, device="cuda")
    y = torch.empty(s.n_dof, dtype=torch.float64, device="cuda")
    A.apply(g["ctrl"], g["young"], prob.nu, ut, y)
    y2 = torch.empty_like(y)
    A.apply(g["ctrl"], g["young"], prob.nu, ut, y2)
    assert torch.equal(y, y2)
    rp = torch.empty(s.n_dof + 1, dtype=torch.int64, device="cuda")
    ci = torch.empty(s.nnz, dtype=torch.int32, device="cuda")
    A.pattern(rp, ci)
    K = torch.sparse_csr_tensor(rp, ci.to(torch.int64), g["vals"], size=(s.n_dof, s.n_dof))
    yc = torch.mv(K, ut)
    assert (torch.linalg.norm(y - yc) / torch.linalg.norm(yc)).item() < 1e-12
    ob = oracle_problem(c)
    vals_ref, _ = As.assemble_lookup(ob["prob"], ob["tabs"], ob["pattern"])
    pt = ob["pattern"]
    Kref = sp.csr_matrix((vals_ref, pt.col_idx(), pt.row_ptr), shape=(s.n_dof, s.n_dof))
    assert rel(y.cpu().numpy(), Kref @ u) < TOL_K


def test_matrix_free_apply_sharded():
    """Each shard's apply gives exactly its rows of the whole problem's apply."""
    from paper_2107_09568_b200 import Assembler
    from synth import draw_uv_seeded
    g = gpu_case(3)
    prob, A = g["prob"], g["A"]
    s = A.sizes
    u, _ = draw_uv_seeded(3, s.n_dof)
    ut = torch.tensor(u, device="cuda")
    y = torch.empty(s.n_dof, dtype=torch.float64, device="cuda")
    A.apply(g["ctrl"], g["young"], prob.nu, ut, y)
    for k in range(3):
        B = Assembler(prob, shard=(3, k))
        z = B.sizes
        yk = torch.empty(z.n_rows, dtype=torch.float64, device="cuda")
        B.apply(g["ctrl"], g["young"], prob.nu, ut, yk)
        assert torch.equal(yk, y[z.row_begin:z.row_begin + z.n_rows]), k


def test_assemble_sensitivity_combined_call():
    """iga_assemble_sensitivity gives the same bits as iga_assemble + iga_sensitivity, with
    device and with (pinned) host u, v."""
    from synth import draw_uv_seeded
    g = gpu_case(2)
    prob, A = g["prob"], g["A"]
    s = A.sizes
    u, v = draw_uv_seeded(2, s.n_dof)
    ut, vt = torch.tensor(u, device="cuda"), torch.tensor(v, device="cuda")
    g1 = torch.empty(s.n_macro_cp * prob.d, dtype=torch.float64, device="cuda")
    A.sensitivity(g["ctrl"], g["young"], prob.nu, ut, vt, g1)
    vals = torch.empty_like(g["vals"])
    g2 = torch.empty_like(g1)
    A.assemble_sensitivity(g["ctrl"], g["young"], prob.nu, ut, vt, vals, g2)
    assert torch.equal(vals, g["vals"]) and torch.equal(g2, g1)
    hu, hv = torch.tensor(u).pin_memory(), torch.tensor(v).pin_memory()
    gh = np.empty(s.n_macro_cp * prob.d)
    A.assemble_sensitivity(g["ctrl"], g["young"], prob.nu, hu.numpy(), hv.numpy(), vals, gh)
    torch.cuda.synchronize()
    assert np.array_equal(gh, g1.cpu().numpy()) and torch.equal(vals, g["vals"])


# ---------------------------------------------------------------------------
# L2 projection with an m-point Gauss rule (iga_set_projection; Eqs. 23-24; NEXT N2)

@pytest.mark.parametrize("c,m,kw", [(1, 4, {}), (1, 6, {}), (2, 4, {}), (2, 5, dict(n_el=(2, 2, 1))),
                                    (4, 5, dict(n_el=(2, 2, 2)))])
def test_l2_projection_parity(c, m, kw):
    """Coefficients, element matrices, K and the sensitivity with the L2 projection of
    m points per direction against the oracle's plain Eqs. 23-24 solve."""
    import dataclasses
    from paper_2107_09568_b200 import Assembler
    from oracle import assemble as As, macro as M, sensitivity as S
    from oracle.dofmap import DofMap, Pattern
    from synth import make_config, draw_uv_seeded
    prob = dataclasses.replace(make_config(c, **kw), n_proj=m)
    # both sides solve the projection (GPU: explicit 1D operator (VᵀWV)⁻¹VᵀW per
    # direction; oracle: the full tensor M_π system): rounding is bounded by
    # κ(M_π)^d·ε, κ(M_π,1D) = 10 at q=2, 35 at q=3 (9.5e-12 in 3D at q=3)
    X1, w1 = M.projection_nodes(m, 1)
    from oracle.bspline import bernstein
    N1 = bernstein(prob.q, X1)
    kappa = np.linalg.cond((N1 * w1) @ N1.T) ** prob.d * 2.0 ** -52
    tol_c, tol_e, tol_k, tol_s = (max(t, 2 * kappa) for t in (TOL_COEF, TOL_ELEM, TOL_K, TOL_SENS))
    A = Assembler(prob)
    A.set_projection(m)
    assert A.projection() == m
    s = A.sizes
    d = prob.d
    dev = torch.device("cuda")
    ctrl = torch.tensor(prob.macro.ctrl, device=dev)
    young = torch.tensor(prob.young, device=dev)
    coef = torch.zeros(s.n_tiles * d * d * s.k_stride, dtype=torch.float64, device=dev)
    A.interpolate(ctrl, young, prob.nu, coef)
    cg = coef.view(s.n_tiles, d * d, s.k_stride)[:, :, :s.n_k].cpu().numpy()
    for t in range(min(prob.n_tiles, 8)):
        ref = M.tile_coefficients(prob, prob.macro.ctrl, t)
        refm = np.transpose(ref, (3, 4, 1, 2, 0)).reshape(d * d, -1)
        assert rel(cg[t], refm) < tol_c, t
    dm = DofMap(prob)
    tabs = As.Tables(prob)
    pt = Pattern(prob, dm, tabs.pairs)
    vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
    local = torch.empty(s.n_local_rows * s.n_tiles * d * d, dtype=torch.float64, device=dev)
    A.assemble(ctrl, young, prob.nu, vals, local)
    ref_vals, ref_local = As.assemble_lookup(prob, tabs, pt)
    L = local.view(s.n_local_rows, s.n_tiles, d, d).permute(1, 0, 2, 3).cpu().numpy()
    for t in range(prob.n_tiles):
        assert rel(L[t], ref_local[t]) < tol_e, t
    assert rel(vals.cpu().numpy(), ref_vals) < tol_k
    u, v = draw_uv_seeded(c, s.n_dof)
    grad = torch.empty(s.n_macro_cp * d, dtype=torch.float64, device=dev)
    A.sensitivity(ctrl, young, prob.nu, torch.tensor(u, device=dev), torch.tensor(v, device=dev), grad)
    got = grad.cpu().numpy().reshape(-1, d)
    ref = S.sensitivity(prob, tabs, pt, u, v)                            # complete gradient
    assert rel(got, ref) < tol_s


def test_projection_errors():
    from paper_2107_09568_b200 import IgaError
    g = gpu_case(2)
    A = g["A"]
    with pytest.raises(IgaError, match="EINVAL"):
        A.set_projection(2)            # m < q+1
    with pytest.raises(IgaError, match="ELIMIT|EINVAL"):
        A.set_projection(7)            # 3D staging exceeds shared memory
    assert A.projection() == 3


# ---------------------------------------------------------------------------
# volume, volume gradient, load vector (NEXT N3; Eqs. 14-19, 53, 66-67)

@pytest.mark.parametrize("c,kw", [(1, {}), (2, {}), (3, dict(n_el=(2, 2, 2))), (4, dict(n_el=(2, 2, 2))),
                                  (2, dict(n_proj=5))])
def test_volume_load_parity(c, kw):
    """V^π, dV^π/dP and the body-force load vector against the oracle."""
    import dataclasses
    from paper_2107_09568_b200 import Assembler
    from oracle import volume as V
    from oracle.dofmap import DofMap
    from synth import make_config
    m = kw.pop("n_proj", 0)
    prob = make_config(c, **kw)
    if m:
        prob = dataclasses.replace(prob, n_proj=m)
    A = Assembler(prob)
    if m:
        A.set_projection(m)
    s = A.sizes
    d = prob.d
    ctrl = torch.tensor(prob.macro.ctrl, device="cuda")
    grad = torch.empty(s.n_macro_cp * d, dtype=torch.float64, device="cuda")
    vol = A.volume(ctrl, grad)
    vref = V.volume_lookup(prob)
    assert abs(vol - vref) < 1e-13 * abs(vref)
    gref = V.volume_gradient(prob)
    assert rel(grad.cpu().numpy().reshape(-1, d), gref) < 1e-12
    dm = DofMap(prob)
    b = np.array([0.5, -1.0, 2.0][:d])
    f = torch.empty(s.n_dof, dtype=torch.float64, device="cuda")
    A.load_vector(ctrl, b, f)
    fref = V.load_vector(prob, dm.node, dm.n_nodes, b)
    assert rel(f.cpu().numpy().reshape(-1, d), fref) < 1e-12
    # shards: volumes and gradients add up, load rows are the whole problem's rows
    if c == 3:
        vs, gs = 0.0, torch.zeros_like(grad)
        for k in range(2):
            B = Assembler(prob, shard=(2, k))
            z = B.sizes
            gk = torch.empty_like(grad)
            vs += B.volume(ctrl, gk)
            gs += gk
            fk = torch.empty(z.n_rows, dtype=torch.float64, device="cuda")
            B.load_vector(ctrl, b, fk)
            assert torch.equal(fk, f[z.row_begin:z.row_begin + z.n_rows])
        assert abs(vs - vol) < 1e-13 * abs(vol)
        assert (torch.linalg.norm(gs - grad) / torch.linalg.norm(grad)).item() < 1e-13


# ---------------------------------------------------------------------------
# NURBS macro map (NEXT N4): the exact rational quarter annulus

@pytest.mark.parametrize("n_el", [(2, 2, 2), (3, 2, 1)])
def test_nurbs_macro_parity(n_el):
    """K, element matrices, the sensitivity and the volume (+ gradient) with a rational
    macro map against the oracle (rational basis, quotient rule, complex step)."""
    from paper_2107_09568_b200 import Assembler
    from oracle import assemble as As, sensitivity as S, volume as V
    from oracle.dofmap import DofMap, Pattern
    from synth import make_config, draw_uv_seeded
    prob = make_config(3, macro_kind="nurbs", n_el=n_el)
    assert prob.macro.weights is not None
    A = Assembler(prob)
    s = A.sizes
    d = 3
    dev = torch.device("cuda")
    ctrl = torch.tensor(prob.macro.ctrl, device=dev)
    young = torch.tensor(prob.young, device=dev)
    vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
    local = torch.empty(s.n_local_rows * s.n_tiles * d * d, dtype=torch.float64, device=dev)
    A.assemble(ctrl, young, prob.nu, vals, local)
    dm = DofMap(prob)
    tabs = As.Tables(prob)
    pt = Pattern(prob, dm, tabs.pairs)
    ref_vals, ref_local = As.assemble_lookup(prob, tabs, pt)
    L = local.view(s.n_local_rows, s.n_tiles, d, d).permute(1, 0, 2, 3).cpu().numpy()
    for t in range(prob.n_tiles):
        assert rel(L[t], ref_local[t]) < TOL_ELEM, t
    assert rel(vals.cpu().numpy(), ref_vals) < TOL_K
    u, v = draw_uv_seeded(3, s.n_dof)
    grad = torch.empty(s.n_macro_cp * d, dtype=torch.float64, device=dev)
    A.sensitivity(ctrl, young, prob.nu, torch.tensor(u, device=dev), torch.tensor(v, device=dev), grad)
    ref = S.sensitivity(prob, tabs, pt, u, v)
    assert rel(grad.cpu().numpy().reshape(-1, d), ref) < TOL_SENS
    gv = torch.empty_like(grad)
    vol = A.volume(ctrl, gv)
    assert abs(vol - V.volume_lookup(prob)) < 1e-13 * vol
    assert rel(gv.cpu().numpy().reshape(-1, d), V.volume_gradient(prob)) < 1e-12


# ---------------------------------------------------------------------------
# edge cases: one tile, lowest / highest degrees, ragged tile counts, degree-1 maps

def _custom_problem(d, p, q, n_el, tile_el, pm=2, amp=0.05, tile_amp=0.08, seed=7):
    from synth.configs import Problem, macro_box, tile_single
    rng = np.random.default_rng(seed)
    lengths = (2.0, 1.0, 1.0)[:d]
    macro = macro_box(pm, n_el, lengths, rng, amp)
    tile = tile_single(p, tile_el, rng, tile_amp)
    prob = Problem(f"edge{d}{p}{q}", d, p, q, 0.3, macro, tile, [], None, tuple(n_el), 0)
    prob.young = rng.uniform(0.5, 2.0, size=int(np.prod(n_el)))
    return prob


@pytest.mark.parametrize("d,p,q,n_el,tile_el,pm", [
    (2, 2, 2, (1, 1), (3, 3), 2),          # a single tile
    (3, 2, 2, (1, 1, 1), (2, 2, 2), 2),    # a single 3D tile
    (2, 2, 0, (3, 2), (3, 3), 2),          # q = 0: n_k = d² (one K3 chunk, tail only)
    (3, 2, 1, (3, 1, 2), (2, 2, 2), 2),    # q = 1
    (3, 2, 0, (2, 2, 1), (2, 2, 2), 2),    # 3D q = 0 (one node per tile: K5b register path, n_π = 1)
    (2, 3, 4, (2, 2), (2, 3), 3),          # q = 4 (max), p = 3, (q+1)^d = 25
    (3, 1, 2, (5, 3, 1), (3, 2, 2), 1),    # p = 1 tiles and a degree-1 macro map; 15 tiles (ragged N-block)
    (2, 4, 3, (9, 2), (2, 2), 2),          # p = 4 (max), 18 tiles = one full 2D N-block
])
def test_edge_case_parity(d, p, q, n_el, tile_el, pm):
    """K, element matrices and the sensitivity against the oracle on edge configurations."""
    from paper_2107_09568_b200 import Assembler
    from oracle import assemble as As, sensitivity as S
    from oracle.dofmap import DofMap, Pattern
    from synth import draw_uv_seeded
    prob = _custom_problem(d, p, q, n_el, tile_el, pm)
    A = Assembler(prob)
    s = A.sizes
    dev = torch.device("cuda")
    ctrl = torch.tensor(prob.macro.ctrl, device=dev)
    young = torch.tensor(prob.young, device=dev)
    vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
    local = torch.empty(s.n_local_rows * s.n_tiles * d * d, dtype=torch.float64, device=dev)
    A.assemble(ctrl, young, prob.nu, vals, local)
    dm = DofMap(prob)
    tabs = As.Tables(prob)
    pt = Pattern(prob, dm, tabs.pairs)
    rp = torch.empty(s.n_dof + 1, dtype=torch.int64, device=dev)
    ci = torch.empty(s.nnz, dtype=torch.int32, device=dev)
    A.pattern(rp, ci)
    assert np.array_equal(rp.cpu().numpy(), pt.row_ptr) and np.array_equal(ci.cpu().numpy(), pt.col_idx())
    ref_vals, ref_local = As.assemble_lookup(prob, tabs, pt)
    L = local.view(s.n_local_rows, s.n_tiles, d, d).permute(1, 0, 2, 3).cpu().numpy()
    kappa = 35.0 ** d * 2.0 ** -52 * 4 if q >= 3 else 0.0   # κ(V1)^d rounding of the interpolation inverse
    for t in range(prob.n_tiles):
        assert rel(L[t], ref_local[t]) < max(TOL_ELEM, kappa), t
    assert rel(vals.cpu().numpy(), ref_vals) < max(TOL_K, kappa)
    u, v = draw_uv_seeded(11, s.n_dof)
    grad = torch.empty(s.n_macro_cp * d, dtype=torch.float64, device=dev)
    A.sensitivity(ctrl, young, prob.nu, torch.tensor(u, device=dev), torch.tensor(v, device=dev), grad)
    ref = S.sensitivity(prob, tabs, pt, u, v)
    assert rel(grad.cpu().numpy().reshape(-1, d), ref) < max(TOL_SENS, kappa)
    y = torch.empty(s.n_dof, dtype=torch.float64, device=dev)
    A.apply(ctrl, young, prob.nu, torch.tensor(u, device=dev), y)
    import scipy.sparse as sp
    Kref = sp.csr_matrix((ref_vals, pt.col_idx(), pt.row_ptr), shape=(s.n_dof, s.n_dof))
    assert rel(y.cpu().numpy(), Kref @ u) < max(TOL_K, kappa)


@pytest.mark.parametrize("c,kw", [(2, {}), (3, dict(n_el=(4, 2, 2)))])
def test_sensitivity_bitwise_deterministic(c, kw):
    """g is bitwise reproducible run to run (no atomics anywhere; the split-K partials of
    small problems are summed in segment order), and the one-call step gives the same bits."""
    from paper_2107_09568_b200 import Assembler
    from synth import make_config, draw_uv_seeded
    prob = make_config(c, **kw)
    A = Assembler(prob)
    s = A.sizes
    d = prob.d
    dev = torch.device("cuda")
    ctrl = torch.tensor(prob.macro.ctrl, device=dev)
    young = torch.tensor(prob.young, device=dev)
    u, v = (torch.tensor(x, device=dev) for x in draw_uv_seeded(c + 90, s.n_dof))
    gs = []
    for _ in range(3):
        g = torch.empty(s.n_macro_cp * d, dtype=torch.float64, device=dev)
        A.sensitivity(ctrl, young, prob.nu, u, v, g)
        gs.append(g)
    vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
    g2 = torch.empty_like(gs[0])
    A.assemble_sensitivity(ctrl, young, prob.nu, u, v, vals, g2)
    torch.cuda.synchronize()
    assert torch.equal(gs[0], gs[1]) and torch.equal(gs[0], gs[2]) and torch.equal(gs[0], g2)


@pytest.mark.parametrize("d,q,n_el,tile_el,split", [
    (3, 1, (2, 2, 2), (5, 5, 5), True),      # 343-point 3D tile patch: K5x + K5a, split-K
    (3, 1, (37, 8, 4), (5, 5, 5), False),    # 1184 tiles = 148 N-blocks: K5x + K5a, one segment
    (2, 2, (3, 2), (13, 13), True),          # 225-point 2D tile patch
    (2, 1, (74, 32), (13, 13), False),       # 2368 tiles = 148 2D N-blocks
])
def test_sensitivity_k5x_k5a_fallback(d, q, n_el, tile_el, split):
    """Tile patches too large for K5g's u/v staging take the K5x + K5a route (X̃ through
    HBM, incl. the column-split refusal guard): complete gradient against the oracle."""
    from paper_2107_09568_b200 import Assembler
    from oracle import assemble as As
    from oracle.dofmap import DofMap, Pattern
    from synth import draw_uv_seeded
    prob = _custom_problem(d, 2, q, n_el, tile_el, 2)
    A = Assembler(prob)
    s = A.sizes
    assert s.sens_path & 1 == 0, "expected the K5x + K5a route"
    assert ((s.sens_path >> 8) > 1) == split
    dev = torch.device("cuda")
    ctrl = torch.tensor(prob.macro.ctrl, device=dev)
    young = torch.tensor(prob.young, device=dev)
    u, v = draw_uv_seeded(21, s.n_dof)
    grad = torch.empty(s.n_macro_cp * d, dtype=torch.float64, device=dev)
    A.set_profiling(True)
    A.sensitivity(ctrl, young, prob.nu, torch.tensor(u, device=dev), torch.tensor(v, device=dev), grad)
    _, n = A.kernel_times()
    assert n[7] >= 1 and n[3] >= 1                                      # K5x and K5a ran
    dm = DofMap(prob)
    tabs = As.Tables(prob)
    pt = Pattern(prob, dm, tabs.pairs)
    parts = PT.run(PT.w_sensitivity, PT.tile_chunks(prob.n_tiles, 16), prob=prob, tabs=tabs, pattern=pt, u=u, v=v)
    ref = np.sum(parts, axis=0)
    got = grad.cpu().numpy().reshape(-1, d)
    assert rel(got, ref) < TOL_SENS, rel(got, ref)
