"""Product-space ILP (P) for two closed triangle meshes.

The reference ships only the behavioural contract for this module
("[MODULE] product_space"); there is no
reference implementation, so this builder defines the instance that both
the CPU oracle and the B200 path consume.

Conventions:
  * ext(X) = 3 cyclic rotations of every oriented face, 6 two-vertex
    triples per undirected edge (aab, aba, baa, abb, bab, bba) and one
    (v, v, v) per vertex.
  * P = ext(M) x ext(N) minus both-degenerate pairs, quotiented by the
    simultaneous cyclic rotation; each class is stored in its
    lexicographically smallest rotation.
  * A_boundary: one row per undirected product edge, +1 for a boundary edge
    that runs from the lexicographically smaller vertex pair to the larger,
    -1 otherwise; rhs 0.  A^M / A^N: one row per face, sum of the product
    triangles whose M- (N-) side is a rotation of it equals 1.
  * Costs: Eq. (2), c_p = sum_v (A^M_{m_v} + A^N_{n_v}) ||F_{m_v} - F_{n_v}||
    with Meyer mixed vertex areas.

Variable numbering.  The reference's averaging passes are Gauss-Seidel
sweeps in variable order (kernels.py:194-269), so the numbering fixes the
dependency DAG the B200 exact-MMA kernel schedules by levels.  Product
triangles are numbered by a "row colour": every A^M and A^N row receives
each colour at most once (a Latin-square colouring of the face pairs plus
one colour per degenerate element), so both projection-row chains advance
one level per colour; a greedy colouring of every row's variables, taken in
that order, then fixes the numbering (boundary rows and pruning leave the
Latin colours sparse), and the DAG depth stays close to its lower bound,
the longest row.  ``order="natural"`` keeps the enumeration order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# product triangle kinds
TRI_TRI, TRI_EDGE, TRI_VERTEX, EDGE_TRI, VERTEX_TRI = range(5)
KIND_NAMES = ("tri-tri", "tri-edge", "tri-vertex", "edge-tri", "vertex-tri")


@dataclass
class Mesh:
    vertices: np.ndarray  # (V, 3) float64
    faces: np.ndarray  # (T, 3) int64, counterclockwise

    @property
    def num_vertices(self) -> int:
        return len(self.vertices)

    @property
    def num_faces(self) -> int:
        return len(self.faces)

    def edges(self) -> np.ndarray:
        """Undirected edges (a < b), sorted lexicographically."""
        f = self.faces
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
        e = np.sort(e, axis=1)
        return np.unique(e, axis=0)


def icosphere(subdivisions: int) -> Mesh:
    """Unit icosahedron refined ``subdivisions`` times (1-to-4 split)."""
    t = (1.0 + 5.0 ** 0.5) / 2.0
    v = np.array(
        [[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t],
         [0, -1, -t], [0, 1, -t], [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]],
        dtype=np.float64,
    )
    f = np.array(
        [[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4],
         [11, 10, 2], [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8],
         [3, 8, 9], [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]],
        dtype=np.int64,
    )
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    verts = [tuple(x) for x in v]
    for _ in range(subdivisions):
        mid = {}
        new_faces = []

        def midpoint(a, b):
            key = (min(a, b), max(a, b))
            if key not in mid:
                p = (np.asarray(verts[a]) + np.asarray(verts[b])) / 2.0
                p /= np.linalg.norm(p)
                mid[key] = len(verts)
                verts.append(tuple(p))
            return mid[key]

        for a, b, c in f.tolist():
            ab, bc, ca = midpoint(a, b), midpoint(b, c), midpoint(c, a)
            new_faces += [[a, ab, ca], [b, bc, ab], [c, ca, bc], [ab, bc, ca]]
        f = np.asarray(new_faces, dtype=np.int64)
    return Mesh(np.asarray(verts, dtype=np.float64), f)


def deform(mesh: Mesh, seed: int, amplitude: float = 0.25, modes: int = 6) -> Mesh:
    """Smooth random non-rigid deformation (sum of low-frequency bumps)."""
    rng = np.random.default_rng(seed)
    x = mesh.vertices
    disp = np.zeros_like(x)
    for _ in range(modes):
        k = rng.standard_normal(3) * 1.5
        phase = rng.uniform(0, 2 * np.pi)
        direction = rng.standard_normal(3)
        disp += np.sin(x @ k + phase)[:, None] * direction[None, :]
    disp *= amplitude / max(1e-12, np.abs(disp).max())
    return Mesh(x + disp, mesh.faces.copy())


def mixed_vertex_areas(mesh: Mesh) -> np.ndarray:
    """Meyer et al. mixed areas: Voronoi cotangent areas on
    non-obtuse triangles, area/2 at an obtuse corner and area/4 elsewhere."""
    x = mesh.vertices
    f = mesh.faces
    out = np.zeros(len(x))
    p = [x[f[:, k]] for k in range(3)]
    cross = np.cross(p[1] - p[0], p[2] - p[0])
    area = 0.5 * np.linalg.norm(cross, axis=1)
    if (area <= 0).any():
        raise ValueError("degenerate triangle")
    for k in range(3):
        a, b, c = p[k], p[(k + 1) % 3], p[(k + 2) % 3]
        # angle at b and c -> cot; Voronoi share of vertex a
        ab, ac = b - a, c - a
        ba, bc = a - b, c - b
        ca, cb = a - c, b - c
        cot_b = np.einsum("ij,ij->i", ba, bc) / np.linalg.norm(np.cross(ba, bc), axis=1)
        cot_c = np.einsum("ij,ij->i", ca, cb) / np.linalg.norm(np.cross(ca, cb), axis=1)
        vor = (np.einsum("ij,ij->i", ac, ac) * cot_b + np.einsum("ij,ij->i", ab, ab) * cot_c) / 8.0
        dot_a = np.einsum("ij,ij->i", ab, ac)
        dot_b = np.einsum("ij,ij->i", ba, bc)
        dot_c = np.einsum("ij,ij->i", ca, cb)
        obtuse_any = (dot_a < 0) | (dot_b < 0) | (dot_c < 0)
        share = np.where(~obtuse_any, vor, np.where(dot_a < 0, area / 2.0, area / 4.0))
        np.add.at(out, f[:, k], share)
    return out


def random_features(n: int, dim: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal((n, dim))


def smooth_features(mesh_ref: Mesh, dim: int, seed: int, noise: float = 0.0,
                    noise_seed: int = 0) -> np.ndarray:
    """Random Fourier features of reference positions (correspondence-aware
    synthetic descriptors), plus optional per-vertex noise."""
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((3, dim)) * 2.0
    b = rng.uniform(0, 2 * np.pi, dim)
    feats = np.cos(mesh_ref.vertices @ w + b)
    if noise:
        feats = feats + noise * np.random.default_rng(noise_seed).standard_normal(feats.shape)
    return feats


def geodesic_sphere(freq: int) -> Mesh:
    """Class-I geodesic sphere: every icosahedron face cut into a freq x freq
    triangular grid, projected to the unit sphere (20 freq^2 faces: 500 at
    freq 5, 980 at freq 7; genus 0, consistently outward-oriented)."""
    ico = icosphere(0)
    key, verts, faces = {}, [], []

    def vid(p):
        p = p / np.linalg.norm(p)
        k = tuple(np.round(p, 9))
        if k not in key:
            key[k] = len(verts)
            verts.append(p)
        return key[k]

    for a, b, c in ico.faces.tolist():
        A, B, C = ico.vertices[a], ico.vertices[b], ico.vertices[c]
        idx = {(i, j): vid((i * A + j * B + (freq - i - j) * C) / freq)
               for i in range(freq + 1) for j in range(freq + 1 - i)}
        for i in range(freq):
            for j in range(freq - i):
                faces.append([idx[i, j], idx[i + 1, j], idx[i, j + 1]])
                if i + j < freq - 1:
                    faces.append([idx[i + 1, j], idx[i + 1, j + 1], idx[i, j + 1]])
    return Mesh(np.asarray(verts, dtype=np.float64), np.asarray(faces, dtype=np.int64))


def humanoid(mesh: Mesh) -> Mesh:
    """Radial map of a sphere to a humanoid-like genus-0 body: flattened
    torso with five Gaussian lobes (head, two arms, two legs)."""
    x = mesh.vertices
    dirs = np.array([[0, 1, 0], [0.95, 0.3, 0], [-0.95, 0.3, 0], [0.35, -0.94, 0], [-0.35, -0.94, 0]])
    dirs = dirs / np.linalg.norm(dirs, axis=1, keepdims=True)
    amp = np.array([0.6, 1.1, 1.1, 1.3, 1.3])
    wid = np.array([0.10, 0.05, 0.05, 0.06, 0.06])
    r = 1.0 + (amp[None] * np.exp(-(1.0 - x @ dirs.T) / wid[None])).sum(1)
    y = x * r[:, None]
    y[:, 2] *= 0.5
    return Mesh(y, mesh.faces.copy())


def cotan_laplacian(mesh: Mesh) -> np.ndarray:
    """Dense cotangent stiffness matrix (V x V; meshes here have < 1000 vertices)."""
    x, f = mesh.vertices, mesh.faces
    W = np.zeros((len(x), len(x)))
    for k in range(3):
        i, j, o = f[:, (k + 1) % 3], f[:, (k + 2) % 3], f[:, k]
        u, v = x[i] - x[o], x[j] - x[o]
        cot = np.einsum("ij,ij->i", u, v) / np.linalg.norm(np.cross(u, v), axis=1)
        np.add.at(W, (i, j), 0.5 * cot)
        np.add.at(W, (j, i), 0.5 * cot)
    return np.diag(W.sum(1)) - W


def heat_kernel_signature(mesh: Mesh, dim: int = 16, eigs: int = 60) -> np.ndarray:
    """Spectral descriptors: log heat kernel signature at ``dim`` log-spaced
    times from the first ``eigs`` Laplace-Beltrami eigenpairs (lumped mixed
    areas as mass), area-normalised per time, centred per time, rounded to
    1e-6 so that the last-bit differences of LAPACK/BLAS builds and thread
    counts do not reach the costs (the builder output is hashed bitwise)."""
    L = cotan_laplacian(mesh)
    a = mixed_vertex_areas(mesh)
    s = 1.0 / np.sqrt(a)
    lam, phi = np.linalg.eigh(s[:, None] * L * s[None, :])
    lam, phi = lam[:eigs], (s[:, None] * phi)[:, :eigs]
    ts = np.geomspace(4 * np.log(10) / lam[eigs - 1], 4 * np.log(10) / lam[1], dim)
    h = (phi ** 2) @ np.exp(-lam[:, None] * ts[None])
    h = np.log(h / (a[:, None] * h).sum(0, keepdims=True))
    return np.round(h - h.mean(0), 6)


def knn_allowed(feat_m: np.ndarray, feat_n: np.ndarray, k: int) -> np.ndarray:
    """Symmetric k-NN pruning in descriptor space: vertex
    pair (i, j) is kept when j is among i's k nearest or i among j's."""
    D = ((feat_m[:, None, :] - feat_n[None, :, :]) ** 2).sum(-1)
    al = np.zeros(D.shape, bool)
    nm = np.argsort(D, 1, kind="stable")[:, :k]
    nn = np.argsort(D, 0, kind="stable")[:k].T
    al[np.repeat(np.arange(D.shape[0]), k), nm.ravel()] = True
    al[nn.ravel(), np.repeat(np.arange(D.shape[1]), k)] = True
    return al


def _edge_triples(edges: np.ndarray) -> np.ndarray:
    a, b = edges[:, 0], edges[:, 1]
    pats = [(a, a, b), (a, b, a), (b, a, a), (a, b, b), (b, a, b), (b, b, a)]
    return np.stack([np.stack(p, axis=1) for p in pats], axis=1).reshape(-1, 3)


@dataclass
class ProductSpace:
    m: np.ndarray  # (P, 3) M vertex of each corner (canonical rotation)
    n: np.ndarray  # (P, 3) N vertex of each corner
    kind: np.ndarray  # (P,) int8 kind
    face_m: np.ndarray  # (P,) M face id or -1
    face_n: np.ndarray  # (P,) N face id or -1
    costs: np.ndarray  # (P,) float64
    row_ptr: np.ndarray  # CSR over rows: boundary rows, then A^M, then A^N
    row_var: np.ndarray
    row_coef: np.ndarray
    row_rhs: np.ndarray
    num_boundary_rows: int
    num_vm: int
    num_vn: int

    @property
    def num_variables(self) -> int:
        return len(self.costs)

    @property
    def num_rows(self) -> int:
        return len(self.row_rhs)

    def rows(self):
        """Rows as (variables, coefficients, rhs) tuples (reference layout)."""
        out = []
        for r in range(self.num_rows):
            lo, hi = self.row_ptr[r], self.row_ptr[r + 1]
            out.append((self.row_var[lo:hi], self.row_coef[lo:hi], int(self.row_rhs[r])))
        return out


def _canonical_rotation(m, n):
    """Rotate each corner triple to its lexicographically smallest rotation."""
    P = len(m)
    keys = []
    for k in range(3):
        idx = [(k + j) % 3 for j in range(3)]
        keys.append(np.stack([m[:, idx[0]], n[:, idx[0]], m[:, idx[1]], n[:, idx[1]],
                              m[:, idx[2]], n[:, idx[2]]], axis=1))
    best = np.zeros(P, dtype=np.int64)
    cur = keys[0].copy()
    rows = np.arange(P)
    for k in (1, 2):
        cand = keys[k]
        diff = cand != cur
        first = np.argmax(diff, axis=1)
        less = diff.any(axis=1) & (cand[rows, first] < cur[rows, first])
        best = np.where(less, k, best)
        cur = np.where(less[:, None], cand, cur)
    rot = (np.arange(3)[None, :] + best[:, None]) % 3
    return np.take_along_axis(m, rot, 1), np.take_along_axis(n, rot, 1)


def build_product_space(M: Mesh, N: Mesh, feat_m: np.ndarray, feat_n: np.ndarray,
                        order: str = "auto", allowed: np.ndarray | None = None,
                        order_seed: int = 2, colouring=None) -> ProductSpace:
    """Enumerate P, order the variables, assemble rows and Eq. (2) costs.

    ``allowed`` (optional, bool (|V_M|, |V_N|)) keeps only product triangles
    whose three vertex pairs are all allowed (k-NN / coarse-to-fine pruning,
    SPEC.md:489-500).

    ``order``: "greedy" (default, "auto"): the Latin-square colour order
    refined by a greedy row colouring (dm_row_colouring), numbering by the
    refined colour — the exact passes' DAG depth is then bounded by the
    number of colours: C4 1,665 -> 370 levels, C3 752 -> 199 (on a pruned
    space most Latin colours are sparse and the rows chain through many of
    them), C2 4,119 -> 4,064, C1 1,158 -> 1,016; "colour" (the Latin-square
    colours alone), "natural" (enumeration order).  ``colouring`` (ProductSpace -> colours) replaces
    the native ``row_colouring`` (bench.py's CPU arm passes the oracle's C
    copy, so it builds the same instance without the product library).
    """
    if order == "auto":
        order = "greedy"
    if feat_m.shape[1] != feat_n.shape[1]:
        raise ValueError("feature dimension mismatch")
    FM, FN = M.faces, N.faces
    TM, TN = len(FM), len(FN)
    EM, EN = M.edges(), N.edges()
    E6M, E6N = _edge_triples(EM), _edge_triples(EN)
    VM, VN = M.num_vertices, N.num_vertices
    T = max(TM, TN)
    rotN = np.stack([FN[:, [(k + s) % 3 for k in range(3)]] for s in range(3)], 1)  # (TN,3,3)
    # colour shifts: a random Latin square for the face pairs and a per-face
    # cyclic shift of each degenerate class (a bijection inside every A^M /
    # A^N row), which keeps boundary rows from chaining same-colour
    # variables of neighbouring faces
    rng = np.random.default_rng(order_seed)
    piM, piN = rng.permutation(T), rng.permutation(T)
    shift_te, shift_tv = rng.integers(0, len(E6N), TM), rng.integers(0, VN, TM)
    shift_et, shift_vt = rng.integers(0, len(E6M), TN), rng.integers(0, VM, TN)

    parts = []  # (m, n, kind, face_m, face_n, colour)
    # tri-tri: M face f in stored rotation, N face g rotated by s
    f, g, s = np.meshgrid(np.arange(TM), np.arange(TN), np.arange(3), indexing="ij")
    f, g, s = f.ravel(), g.ravel(), s.ravel()
    parts.append((FM[f], rotN[g, s], TRI_TRI, f, g, 3 * ((piM[f] + piN[g]) % T) + s))
    # tri-edge / tri-vertex: M face, N degenerate element
    f, t = np.meshgrid(np.arange(TM), np.arange(len(E6N)), indexing="ij")
    f, t = f.ravel(), t.ravel()
    parts.append((FM[f], E6N[t], TRI_EDGE, f, np.full_like(f, -1), 3 * T + (t + shift_te[f]) % len(E6N)))
    f, v = np.meshgrid(np.arange(TM), np.arange(VN), indexing="ij")
    f, v = f.ravel(), v.ravel()
    parts.append((FM[f], np.stack([v, v, v], 1), TRI_VERTEX, f, np.full_like(f, -1),
                  3 * T + len(E6N) + (v + shift_tv[f]) % VN))
    # edge-tri / vertex-tri: M degenerate element, N face g in stored rotation
    t, g = np.meshgrid(np.arange(len(E6M)), np.arange(TN), indexing="ij")
    t, g = t.ravel(), g.ravel()
    parts.append((E6M[t], FN[g], EDGE_TRI, np.full_like(g, -1), g, 3 * T + (t + shift_et[g]) % len(E6M)))
    v, g = np.meshgrid(np.arange(VM), np.arange(TN), indexing="ij")
    v, g = v.ravel(), g.ravel()
    parts.append((np.stack([v, v, v], 1), FN[g], VERTEX_TRI, np.full_like(g, -1), g,
                  3 * T + len(E6M) + (v + shift_vt[g]) % VM))

    m = np.concatenate([p[0] for p in parts]).astype(np.int64)
    n = np.concatenate([p[1] for p in parts]).astype(np.int64)
    kind = np.concatenate([np.full(len(p[0]), p[2], np.int8) for p in parts])
    face_m = np.concatenate([p[3] for p in parts]).astype(np.int64)
    face_n = np.concatenate([p[4] for p in parts]).astype(np.int64)
    colour = np.concatenate([p[5] for p in parts]).astype(np.int64)

    if allowed is not None:
        keep = allowed[m, n].all(axis=1)
        m, n, kind, face_m, face_n, colour = (a[keep] for a in (m, n, kind, face_m, face_n, colour))

    if order in ("colour", "greedy"):
        perm = np.lexsort((np.arange(len(m)), colour))
    elif order == "natural":
        perm = np.arange(len(m))
    else:
        raise ValueError(f"unknown order {order!r}")
    m, n, kind, face_m, face_n = m[perm], n[perm], kind[perm], face_m[perm], face_n[perm]
    m, n = _canonical_rotation(m, n)
    out = _assemble(M, N, feat_m, feat_n, m, n, kind, face_m, face_n)
    if order == "greedy":
        perm = np.lexsort((np.arange(out.num_variables), (colouring or row_colouring)(out)))
        out = _assemble(M, N, feat_m, feat_n, m[perm], n[perm], kind[perm], face_m[perm], face_n[perm])
    return out


def row_colouring(p: ProductSpace) -> np.ndarray:
    """Greedy row colouring of the variables in index order (dm_row_colouring)."""
    from . import _native

    colour = np.empty(p.num_variables, np.int64)
    rp = np.ascontiguousarray(p.row_ptr, dtype=np.int64)
    rv = np.ascontiguousarray(p.row_var, dtype=np.int64)
    _native.check(_native.load().dm_row_colouring(p.num_variables, p.num_rows, rp.ctypes.data, rv.ctypes.data,
                                                  colour.ctypes.data), "row colouring")
    return colour


def _assemble(M: Mesh, N: Mesh, feat_m, feat_n, m, n, kind, face_m, face_n) -> ProductSpace:
    """Eq. (2) costs and the rows of numbered product triangles (canonical
    rotation already applied)."""
    VM, VN = M.num_vertices, N.num_vertices
    TM, TN = len(M.faces), len(N.faces)
    P = len(m)

    # Eq. (2) costs, summed corner by corner on the canonical rotation
    area_m, area_n = mixed_vertex_areas(M), mixed_vertex_areas(N)
    costs = np.zeros(P)
    for k in range(3):
        dist = np.linalg.norm(feat_m[m[:, k]] - feat_n[n[:, k]], axis=1)
        costs = costs + (area_m[m[:, k]] + area_n[n[:, k]]) * dist

    # boundary rows: group the 3P oriented product-edge incidences
    pid = m * VN + n  # vertex-pair ids
    src = pid.ravel()
    dst = pid[:, [1, 2, 0]].ravel()
    var = np.repeat(np.arange(P, dtype=np.int64), 3)
    lo_, hi_ = np.minimum(src, dst), np.maximum(src, dst)
    sign = np.where(src < dst, 1, -1).astype(np.int64)
    key = lo_ * (VM * VN) + hi_
    o = np.lexsort((var, key))
    key, var_s, sign_s = key[o], var[o], sign[o]
    starts = np.flatnonzero(np.concatenate([[True], key[1:] != key[:-1]]))
    nb = len(starts)
    b_ptr = np.concatenate([starts, [len(key)]]).astype(np.int64)

    # projection rows
    def proj(face, nf):
        sel = np.flatnonzero(face >= 0)
        oo = np.lexsort((sel, face[sel]))
        sel = sel[oo]
        cnt = np.bincount(face[sel], minlength=nf)
        return sel, np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)

    am_var, am_ptr = proj(face_m, TM)
    an_var, an_ptr = proj(face_n, TN)
    row_var = np.concatenate([var_s, am_var, an_var]).astype(np.int64)
    row_coef = np.concatenate([sign_s, np.ones(len(am_var) + len(an_var), np.int64)])
    row_ptr = np.concatenate([b_ptr[:-1], am_ptr[:-1] + len(var_s),
                              an_ptr + len(var_s) + len(am_var)]).astype(np.int64)
    row_rhs = np.concatenate([np.zeros(nb, np.int64), np.ones(TM + TN, np.int64)])
    return ProductSpace(m, n, kind, face_m, face_n, costs, row_ptr, row_var, row_coef, row_rhs,
                        nb, VM, VN)


def verify_solution(ps: ProductSpace, x: np.ndarray) -> list[int]:
    """Exact integer check of all rows; returns violated rows."""
    x = np.asarray(x, dtype=np.int64)
    lhs = np.add.reduceat(ps.row_coef * x[ps.row_var], ps.row_ptr[:-1]) if ps.num_rows else []
    empty = ps.row_ptr[1:] == ps.row_ptr[:-1]
    lhs = np.where(empty, 0, lhs)
    return np.flatnonzero(lhs != ps.row_rhs).tolist()


def synthetic_pair(config: str, seed: int = 0):
    """Mesh pairs and descriptors of the BASELINE configs.

    'tetra' / 'icosa'  — SPEC acceptance anchors (|P| = 368, ratio ~22);
    'c1'  — icosphere subdiv-1 pair (80 x 80), random 16-D descriptors;
    'c2'  — deformed icosphere subdiv-2 pair (320 x 320), smooth descriptors;
    'c3'  — deformed humanoid-like genus-0 pair (500 x 500), heat kernel
            signatures next to the smooth descriptors (k-NN pruned, see
            ``PRUNING_K``);
    'c4'  — the same at 980 x 980 triangles (the ~1000 x 1000 instance).
    """
    if config in ("c3", "c4"):
        base = geodesic_sphere(5 if config == "c3" else 7)
        body = humanoid(base)
        M = deform(body, seed * 2 + 1)
        N = deform(body, seed * 2 + 2)
        sm = [smooth_features(base, 16, seed, noise=0.3, noise_seed=seed * 2 + s) for s in (1, 2)]
        fm = np.hstack([heat_kernel_signature(M), sm[0]])
        fn = np.hstack([heat_kernel_signature(N), sm[1]])
        return M, N, fm, fn
    if config == "tetra":
        v = np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], np.float64)
        f = np.array([[0, 1, 2], [0, 3, 1], [0, 2, 3], [1, 3, 2]], np.int64)
        M = N = Mesh(v, f)
        fm, fn = random_features(4, 8, seed), random_features(4, 8, seed + 1)
    elif config == "icosa":
        M = N = icosphere(0)
        fm, fn = random_features(12, 8, seed), random_features(12, 8, seed + 1)
    elif config == "c1":
        M = icosphere(1)
        N = icosphere(1)
        fm, fn = random_features(M.num_vertices, 16, seed), random_features(N.num_vertices, 16, seed + 1)
    elif config == "c2":
        base = icosphere(2)
        M = deform(base, seed * 2 + 1)
        N = deform(base, seed * 2 + 2)
        fm = smooth_features(base, 16, seed, noise=0.3, noise_seed=seed * 2 + 1)
        fn = smooth_features(base, 16, seed, noise=0.3, noise_seed=seed * 2 + 2)
    else:
        raise ValueError(f"unknown config {config!r}")
    return M, N, fm, fn


# k of the symmetric k-NN pruning per config (None: full product space)
PRUNING_K = {"c3": 10, "c4": 16}


def synthetic_product_space(config: str, seed: int = 0, colouring=None) -> ProductSpace:
    """The product-space ILP of a BASELINE config, pruned where the config
    says so (C3/C4: k-NN in descriptor space)."""
    M, N, fm, fn = synthetic_pair(config, seed)
    k = PRUNING_K.get(config)
    allowed = knn_allowed(fm, fn, k) if k else None
    return build_product_space(M, N, fm, fn, allowed=allowed, colouring=colouring)
