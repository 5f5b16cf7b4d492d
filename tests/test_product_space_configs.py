"""BASELINE configs C3/C4 (k-NN pruned humanoid-like pairs): mesh, descriptor
and pruning invariants, on the CPU.  Their solver parity is the golden case
``ps_c3`` (real-reference outputs, tests/golden/golden.json) and the
full-size GPU properties on C4 (tests/test_full_size.py)."""

import numpy as np
import pytest

from paper_2310_08230_b200 import product_space as ps


@pytest.mark.parametrize("freq", [1, 2, 5, 7])
def test_geodesic_sphere_is_closed_genus0(freq):
    m = ps.geodesic_sphere(freq)
    assert m.num_faces == 20 * freq * freq
    assert m.num_vertices == 10 * freq * freq + 2
    e = m.edges()
    assert m.num_vertices - len(e) + m.num_faces == 2  # Euler characteristic of a sphere
    f = m.faces
    directed = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
    # consistently oriented closed manifold: each directed edge once, its reverse once
    assert len(np.unique(directed, axis=0)) == len(directed)
    key = {tuple(x) for x in directed.tolist()}
    assert all((b, a) in key for a, b in key)
    x = m.vertices
    n = np.cross(x[f[:, 1]] - x[f[:, 0]], x[f[:, 2]] - x[f[:, 0]])
    assert ((n * x[f].mean(1)).sum(1) > 0).all()  # outward


def test_heat_kernel_signature_is_intrinsic_and_quantised():
    body = ps.humanoid(ps.geodesic_sphere(3))
    h = ps.heat_kernel_signature(body)
    assert h.shape == (body.num_vertices, 16)
    assert np.array_equal(h, np.round(h, 6))
    # rigid motions leave it unchanged (up to the quantisation step)
    q, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((3, 3)))
    moved = ps.Mesh(body.vertices @ q.T + 3.0, body.faces)
    assert np.abs(ps.heat_kernel_signature(moved) - h).max() <= 2e-6


def test_knn_allowed_is_symmetric_union():
    rng = np.random.default_rng(1)
    a, b = rng.standard_normal((30, 4)), rng.standard_normal((25, 4))
    al = ps.knn_allowed(a, b, 3)
    D = ((a[:, None] - b[None]) ** 2).sum(-1)
    for i in range(30):
        assert set(np.argsort(D[i])[:3]) <= set(np.flatnonzero(al[i]))
    for j in range(25):
        assert set(np.argsort(D[:, j])[:3]) <= set(np.flatnonzero(al[:, j]))
    assert al.sum() <= 3 * (30 + 25)


@pytest.mark.parametrize("config", ["c3", "c4"])
def test_pruned_configs_keep_every_face_row_and_ground_truth(config):
    p = ps.synthetic_product_space(config)
    M, N, fm, fn = ps.synthetic_pair(config)
    assert M.num_faces == N.num_faces == (500 if config == "c3" else 980)
    empty = (p.row_ptr[1:] == p.row_ptr[:-1])[p.num_boundary_rows:]
    assert not empty.any()  # every A^M / A^N projection row keeps candidates
    full = len(M.faces) * len(N.faces) * 3
    assert p.num_variables < full // 4  # pruned
    # the identity correspondence (both meshes deform the same body) survives
    # the pruning for (almost) every vertex
    al = ps.knn_allowed(fm, fn, ps.PRUNING_K[config])
    assert al[np.arange(len(al)), np.arange(len(al))].mean() > 0.95
    # and its tri-tri variables are all present
    tt = (p.kind == ps.TRI_TRI) & (p.m == p.n).all(1)  # identity corner map
    gt_faces = np.flatnonzero(al[M.faces, N.faces].all(1))
    assert np.array_equal(np.unique(p.face_m[tt]), gt_faces)


def test_pruned_spaces_are_numbered_by_a_greedy_row_colouring():
    """C3 (pruned): the colour classes are valid (no two variables of a row
    share a colour), the numbering is colour-major, the oracle's C copy of the
    colouring gives the same colours (the CPU arm builds the same instance),
    and the exact passes' depth is within a few levels of the colour count."""
    import numpy as np

    from oracle import clib
    from paper_2310_08230_b200 import product_space as ps

    p = ps.synthetic_product_space("c3", 0)
    col = ps.row_colouring(p)
    assert np.array_equal(col, clib.row_colouring(p))
    for r in range(0, p.num_rows, 97):
        c = col[p.row_var[p.row_ptr[r]:p.row_ptr[r + 1]]]
        assert len(np.unique(c)) == len(c)
    q = ps.synthetic_product_space("c3", 0, colouring=clib.row_colouring)
    assert np.array_equal(q.row_var, p.row_var) and np.array_equal(q.costs, p.costs)
    # the greedy numbering is a fixed point: variables already in colour order
    assert np.array_equal(np.lexsort((np.arange(p.num_variables), col)), np.arange(p.num_variables))


def test_reference_arm_builds_its_instance_without_the_product_library():
    import subprocess
    import sys

    code = ("import bench; bench.oracle_instance('c3', 0); "
            "from paper_2310_08230_b200 import _native; assert _native._lib is None, 'product library loaded'")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    assert r.returncode == 0, r.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("config,latin_depth", [("c3", 752), ("c1", 1158)])
def test_exact_pass_depth_follows_the_colour_count(config, latin_depth):
    """The device level orders of the greedy-numbered spaces: the exact
    passes' DAG depth stays within the split couplings of the colour count,
    well under the Latin-square numbering's ("Numbering of a
    product space")."""
    from paper_2310_08230_b200.dual import init_duals
    from paper_2310_08230_b200.ilp import IlpInstance

    p = ps.synthetic_product_space(config, 0)
    colours = int(ps.row_colouring(p).max()) + 1
    inst = IlpInstance.from_csr(p.costs, p.row_ptr, p.row_var, p.row_coef, p.row_rhs, 128)
    info = init_duals(inst, device="cuda:0").dev.info
    assert info["fw_depth"] == info["bw_depth"]
    assert colours <= info["fw_depth"] <= colours + 16 < latin_depth
