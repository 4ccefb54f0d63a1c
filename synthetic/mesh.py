"""Polyhedral mesh containers and the seeded CUBE mesh family of BASELINE.json.

Recipe:
  * n^3 hexahedra on [0,1]^3 (or an nx x ny x nz box of size (nx,ny,nz)/n),
    vertex (i,j,l) at (i,j,l)*h, id = i + (nx+1)*(j + (ny+1)*l).
  * Quad faces are vertex loops whose right-hand normal is +x/+y/+z; every loop
    starts at its smallest-id vertex.  Faces are numbered x-normal first, then y,
    then z, each lexicographically (i fastest, then j, then l).
  * Cells lexicographic (i fastest); face list (x-,x+,y-,y+,z-,z+) with sign -1
    on the low side and +1 on the high side (sign = +1 iff the loop normal points
    out of the cell).
  * config 3: every vertex with 0<i,j,l<n is moved by U(-0.2h,0.2h)^3 drawn with
    numpy.random.default_rng(seed) in vertex-id order; every non-boundary quad is
    then split into the triangles (v0,v1,v2),(v0,v2,v3), v0 its smallest-id
    vertex (both inherit the quad's orientation).
No method arithmetic lives here.
"""
from dataclasses import dataclass, field
import numpy as np


@dataclass
class PolyMesh:
    xyz: np.ndarray            # [nV,3] float64
    face_ptr: np.ndarray       # [nF+1] int64 (CSR over face_vtx)
    face_vtx: np.ndarray       # vertex loops
    cell_ptr: np.ndarray       # [nK+1] int64 (CSR over cell_face)
    cell_face: np.ndarray      # face ids per cell
    cell_face_sign: np.ndarray # int8, +1 iff loop normal points out of the cell
    face_on_boundary: np.ndarray  # uint8 per face
    cell_ijk: np.ndarray = field(default=None)  # [nK,3] lattice index (structured meshes)
    dims: tuple = (0, 0, 0)
    h: float = 0.0

    @property
    def n_vertices(self):
        return self.xyz.shape[0]

    @property
    def n_faces(self):
        return self.face_ptr.shape[0] - 1

    @property
    def n_cells(self):
        return self.cell_ptr.shape[0] - 1

    def face(self, f):
        return self.face_vtx[self.face_ptr[f]:self.face_ptr[f + 1]]

    def cell_faces(self, K):
        s, e = self.cell_ptr[K], self.cell_ptr[K + 1]
        return self.cell_face[s:e], self.cell_face_sign[s:e]


def hex_mesh(n, dims=None, jitter=0.0, seed=0, triangulate=False):
    """Structured hexahedral mesh with h = 1/n and dims=(nx,ny,nz) cells (default n^3)."""
    nx, ny, nz = dims if dims is not None else (n, n, n)
    h = 1.0 / n
    NX, NY, NZ = nx + 1, ny + 1, nz + 1
    I, J, L = np.meshgrid(np.arange(NX), np.arange(NY), np.arange(NZ), indexing="ij")
    # vertex id order: i fastest -> ravel in Fortran order of (i,j,l)
    ii = I.ravel(order="F"); jj = J.ravel(order="F"); ll = L.ravel(order="F")
    xyz = np.stack([ii * h, jj * h, ll * h], axis=1).astype(np.float64)
    if jitter > 0.0:
        inner = (ii > 0) & (ii < nx) & (jj > 0) & (jj < ny) & (ll > 0) & (ll < nz)
        idx = np.nonzero(inner)[0]
        rng = np.random.default_rng(seed)
        xyz[idx] += rng.uniform(-jitter * h, jitter * h, size=(idx.size, 3))

    def vid(i, j, l):
        return i + NX * (j + NY * l)

    loops = []
    bnd = []
    # x-normal faces: i in 0..nx, j<ny, l<nz
    i, j, l = np.meshgrid(np.arange(NX), np.arange(ny), np.arange(nz), indexing="ij")
    i = i.ravel(order="F"); j = j.ravel(order="F"); l = l.ravel(order="F")
    loops.append(np.stack([vid(i, j, l), vid(i, j + 1, l), vid(i, j + 1, l + 1), vid(i, j, l + 1)], 1))
    bnd.append((i == 0) | (i == nx))
    nfx = i.size
    # y-normal faces
    i, j, l = np.meshgrid(np.arange(nx), np.arange(NY), np.arange(nz), indexing="ij")
    i = i.ravel(order="F"); j = j.ravel(order="F"); l = l.ravel(order="F")
    loops.append(np.stack([vid(i, j, l), vid(i, j, l + 1), vid(i + 1, j, l + 1), vid(i + 1, j, l)], 1))
    bnd.append((j == 0) | (j == ny))
    nfy = i.size
    # z-normal faces
    i, j, l = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(NZ), indexing="ij")
    i = i.ravel(order="F"); j = j.ravel(order="F"); l = l.ravel(order="F")
    loops.append(np.stack([vid(i, j, l), vid(i + 1, j, l), vid(i + 1, j + 1, l), vid(i, j + 1, l)], 1))
    bnd.append((l == 0) | (l == nz))
    quads = np.concatenate(loops, 0)
    qbnd = np.concatenate(bnd, 0)

    # cells
    ci, cj, cl = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ci = ci.ravel(order="F"); cj = cj.ravel(order="F"); cl = cl.ravel(order="F")
    fx = lambda i, j, l: i + NX * (j + ny * l)
    fy = lambda i, j, l: nfx + i + nx * (j + NY * l)
    fz = lambda i, j, l: nfx + nfy + i + nx * (j + ny * l)
    qf = np.stack([fx(ci, cj, cl), fx(ci + 1, cj, cl), fy(ci, cj, cl), fy(ci, cj + 1, cl),
                   fz(ci, cj, cl), fz(ci, cj, cl + 1)], 1)
    qs = np.tile(np.array([-1, 1, -1, 1, -1, 1], dtype=np.int8), (ci.size, 1))
    cell_ijk = np.stack([ci, cj, cl], 1)

    if not triangulate:
        nF = quads.shape[0]
        face_ptr = np.arange(0, 4 * nF + 1, 4, dtype=np.int64)
        face_vtx = quads.ravel().astype(np.int64)
        cell_ptr = np.arange(0, 6 * ci.size + 1, 6, dtype=np.int64)
        return PolyMesh(xyz, face_ptr, face_vtx, cell_ptr, qf.ravel().astype(np.int64),
                        qs.ravel(), qbnd.astype(np.uint8), cell_ijk, (nx, ny, nz), h)

    # split every non-boundary quad along the diagonal through its smallest-id vertex (v0)
    split = ~qbnd
    nq = quads.shape[0]
    nsub = np.where(split, 2, 1)
    first = np.concatenate([[0], np.cumsum(nsub)[:-1]])  # new id of first piece
    nF = int(nsub.sum())
    sizes = np.empty(nF, dtype=np.int64)
    sizes[first] = np.where(split, 3, 4)
    sizes[first[split] + 1] = 3
    face_ptr = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    face_vtx = np.empty(face_ptr[-1], dtype=np.int64)
    # unsplit quads
    u = np.nonzero(~split)[0]
    for c in range(4):
        face_vtx[face_ptr[first[u]] + c] = quads[u, c]
    s = np.nonzero(split)[0]
    for c, src in enumerate((0, 1, 2)):
        face_vtx[face_ptr[first[s]] + c] = quads[s, src]
    for c, src in enumerate((0, 2, 3)):
        face_vtx[face_ptr[first[s] + 1] + c] = quads[s, src]
    fbnd = np.zeros(nF, dtype=np.uint8)
    fbnd[first[u]] = 1
    # cells: replace each quad by its pieces, keeping sign
    cnt = nsub[qf]                       # [nK,6]
    per_cell = cnt.sum(1)
    cell_ptr = np.concatenate([[0], np.cumsum(per_cell)]).astype(np.int64)
    cell_face = np.empty(cell_ptr[-1], dtype=np.int64)
    cell_sign = np.empty(cell_ptr[-1], dtype=np.int8)
    pos = cell_ptr[:-1].copy()
    for c in range(6):
        q = qf[:, c]
        cell_face[pos] = first[q]
        cell_sign[pos] = qs[:, c]
        pos += 1
        two = nsub[q] == 2
        cell_face[pos[two]] = first[q[two]] + 1
        cell_sign[pos[two]] = qs[two, c]
        pos[two] += 1
    return PolyMesh(xyz, face_ptr, face_vtx, cell_ptr, cell_face, cell_sign, fbnd,
                    cell_ijk, (nx, ny, nz), h)


def mark_neumann(mesh, sides=("x1", "y1"), tol=1e-9):
    """Input recipe of the paper's numerical setting ("Neumann boundary conditions on two
    faces of the cube and homogeneous Dirichlet on the other ones"): boundary faces lying on the
    named sides of [0,1]^3 ("x0", "x1", "y0", ...) get face_on_boundary = 2 (Neumann), the other
    boundary faces keep 1 (Dirichlet).  Returns a new mesh; nothing else changes."""
    import copy
    fb = np.array(mesh.face_on_boundary, dtype=np.uint8).copy()
    for f in np.nonzero(fb)[0]:
        X = mesh.xyz[mesh.face(f)]
        for sd in sides:
            a, v = "xyz".index(sd[0]), float(sd[1])
            if np.all(np.abs(X[:, a] - v) < tol):
                fb[f] = 2
    out = copy.copy(mesh)          # keeps attributes set outside the dataclass fields (generators)
    out.face_on_boundary = fb
    return out


def box_partition(mesh, sub):
    """Subdomain id per cell for a box partition with `sub`=(sx,sy,sz) cells per subdomain.

    Subdomains are numbered lexicographically (x fastest) over the subdomain grid.
    """
    sx, sy, sz = sub
    nx, ny, nz = mesh.dims
    gx, gy, gz = nx // sx, ny // sy, nz // sz
    c = mesh.cell_ijk
    return ((c[:, 0] // sx) + gx * ((c[:, 1] // sy) + gy * (c[:, 2] // sz))).astype(np.int32), (gx, gy, gz)


# ------------------------------------------------------------------ CVT (Voronoi) meshes, SURVEY f4
def _voronoi_cells(P):
    """Bounded Voronoi tessellation of the unit cube for generators P [N,3] (scipy.spatial.Voronoi
    of P and its mirror images across the 6 faces: the cells of P are exactly clipped by the cube).
    Returns (vertices [nV,3], faces [list of (loop, cell_a, cell_b)] with cell_b = -1 on the
    boundary, loop ordered counter-clockwise about the normal pointing from cell_a to cell_b)."""
    from scipy.spatial import Voronoi
    N = P.shape[0]
    mirrors = [P]
    for d in range(3):
        for w in (0.0, 1.0):
            Q = P.copy()
            Q[:, d] = 2 * w - Q[:, d]
            mirrors.append(Q)
    A = np.concatenate(mirrors, 0)
    vor = Voronoi(A)
    V = vor.vertices.copy()
    # refine every used vertex as the point equidistant from all generators whose cells meet there
    # (least squares over the bisector planes): Qhull's coordinates of nearly degenerate vertices
    # are only ~1e-9 accurate, which would leave faces non-planar at that level
    gens = {}
    for (a, b), rv in zip(vor.ridge_points, vor.ridge_vertices):
        if a >= N and b >= N:
            continue
        for v in rv:
            if v >= 0:
                gens.setdefault(v, set()).update((int(a), int(b)))
    for v, g in gens.items():
        g = sorted(g)
        p0 = A[g[0]]
        M = 2.0 * (A[g[1:]] - p0)
        rhs = (A[g[1:]] ** 2).sum(1) - (p0 ** 2).sum()
        V[v] = np.linalg.lstsq(M, rhs, rcond=None)[0]
    V[np.abs(V) < 1e-12] = 0.0
    V[np.abs(V - 1.0) < 1e-12] = 1.0
    faces = []
    for (a, b), rv in zip(vor.ridge_points, vor.ridge_vertices):
        if a >= N and b >= N:
            continue
        if a >= N:
            a, b = b, a
        rv = [v for v in rv if v >= 0]
        if len(rv) < 3:
            continue
        nrm = A[b] - A[a]
        nrm /= np.linalg.norm(nrm)
        X = V[rv]
        c = X.mean(0)
        t1 = X[0] - c
        t1 -= (t1 @ nrm) * nrm
        t1 /= np.linalg.norm(t1)
        t2 = np.cross(nrm, t1)
        ang = np.arctan2((X - c) @ t2, (X - c) @ t1)
        loop = [rv[i] for i in np.argsort(ang)]
        faces.append((loop, int(a), int(b) if b < N else -1))
    return V, faces


def _cell_centroids(V, faces, N):
    vol = np.zeros(N); m1 = np.zeros((N, 3))
    apex = np.zeros((N, 3)); cnt = np.zeros(N)
    for loop, a, b in faces:
        for cidx in (a, b):
            if cidx >= 0:
                apex[cidx] += V[loop].sum(0); cnt[cidx] += len(loop)
    apex /= cnt[:, None]
    for loop, a, b in faces:
        for cidx, sgn in ((a, 1.0), (b, -1.0)):
            if cidx < 0:
                continue
            p0 = V[loop[0]]
            for i in range(1, len(loop) - 1):
                p1, p2 = V[loop[i]], V[loop[i + 1]]
                v6 = sgn * np.dot(p0 - apex[cidx], np.cross(p1 - apex[cidx], p2 - apex[cidx]))
                vol[cidx] += v6 / 6
                m1[cidx] += v6 / 6 * (apex[cidx] + p0 + p1 + p2) / 4
    return m1 / vol[:, None], vol


def cvt_mesh(m, seed=0, lloyd=20):
    """CVT mesh of [0,1]^3 with m^3 cells (the paper's CVT family): generators
    drawn by numpy.random.default_rng(seed).uniform(0, 1, (m^3, 3)), `lloyd` Lloyd iterations
    (generators -> centroids of their bounded Voronoi cells), then the bounded Voronoi cells.
    Vertices are the Voronoi vertices used by the cells (coordinates within 1e-12 of the cube
    faces snapped onto them); faces are the ridges (planar convex polygons), interior ones stored
    once, loops counter-clockwise about the normal out of their first cell (sign +1 there, -1 in
    the neighbour); boundary faces are the ridges towards mirror images."""
    rng = np.random.default_rng(seed)
    N = m ** 3
    P = rng.uniform(0.0, 1.0, (N, 3))
    for _ in range(lloyd):
        V, faces = _voronoi_cells(P)
        P, _ = _cell_centroids(V, faces, N)
    V, faces = _voronoi_cells(P)
    used = sorted({v for loop, _, _ in faces for v in loop})
    remap = {v: i for i, v in enumerate(used)}
    xyz = V[used].astype(np.float64)
    face_ptr = [0]; face_vtx = []; fb = []
    cell_faces = [[] for _ in range(N)]
    for f, (loop, a, b) in enumerate(faces):
        face_vtx += [remap[v] for v in loop]
        face_ptr.append(len(face_vtx))
        fb.append(1 if b < 0 else 0)
        cell_faces[a].append((f, 1))
        if b >= 0:
            cell_faces[b].append((f, -1))
    cell_ptr = np.concatenate([[0], np.cumsum([len(c) for c in cell_faces])]).astype(np.int64)
    cell_face = np.array([f for c in cell_faces for f, _ in c], dtype=np.int64)
    cell_sign = np.array([s for c in cell_faces for _, s in c], dtype=np.int8)
    mesh = PolyMesh(xyz, np.array(face_ptr, dtype=np.int64), np.array(face_vtx, dtype=np.int64), cell_ptr,
                    cell_face, cell_sign, np.array(fb, dtype=np.uint8), None, (0, 0, 0), 1.0 / m)
    mesh.generators = P
    return mesh


def centroid_partition(mesh, grid):
    """Subdomain id per cell for an sx x sy x sz box partition of [0,1]^3 by cell generator (CVT:
    the generator is the cell centroid), numbered lexicographically (x fastest)."""
    sx, sy, sz = grid
    P = mesh.generators
    ix = np.minimum((P[:, 0] * sx).astype(int), sx - 1)
    iy = np.minimum((P[:, 1] * sy).astype(int), sy - 1)
    iz = np.minimum((P[:, 2] * sz).astype(int), sz - 1)
    return (ix + sx * (iy + sy * iz)).astype(np.int32), (sx, sy, sz)


def _voronoi_mesh(P, h):
    """PolyMesh of the bounded Voronoi cells of generators P in [0,1]^3 (see _voronoi_cells)."""
    N = P.shape[0]
    V, faces = _voronoi_cells(P)
    used = sorted({v for loop, _, _ in faces for v in loop})
    remap = {v: i for i, v in enumerate(used)}
    xyz = V[used].astype(np.float64)
    face_ptr = [0]; face_vtx = []; fb = []
    cell_faces = [[] for _ in range(N)]
    for f, (loop, a, b) in enumerate(faces):
        face_vtx += [remap[v] for v in loop]
        face_ptr.append(len(face_vtx))
        fb.append(1 if b < 0 else 0)
        cell_faces[a].append((f, 1))
        if b >= 0:
            cell_faces[b].append((f, -1))
    cell_ptr = np.concatenate([[0], np.cumsum([len(c) for c in cell_faces])]).astype(np.int64)
    cell_face = np.array([f for c in cell_faces for f, _ in c], dtype=np.int64)
    cell_sign = np.array([s for c in cell_faces for _, s in c], dtype=np.int8)
    mesh = PolyMesh(xyz, np.array(face_ptr, dtype=np.int64), np.array(face_vtx, dtype=np.int64), cell_ptr,
                    cell_face, cell_sign, np.array(fb, dtype=np.uint8), None, (0, 0, 0), h)
    mesh.generators = P
    return mesh


def octa_mesh(n):
    """OCTA family (SPEC's reading: a clipped BCC truncated-octahedron tiling): the Voronoi
    cells of the body-centred cubic lattice {(i + 1/4)/n} u {(i + 3/4)/n} (i = 0..n-1 per axis),
    2 n^3 cells; interior cells are 14-faced truncated octahedra (8 hexagons, 6 squares), the
    boundary ones are clipped by the cube."""
    a = (np.arange(n) + 0.25) / n
    b = (np.arange(n) + 0.75) / n
    A = np.stack(np.meshgrid(a, a, a, indexing="ij"), -1).reshape(-1, 3)
    B = np.stack(np.meshgrid(b, b, b, indexing="ij"), -1).reshape(-1, 3)
    return _voronoi_mesh(np.concatenate([A, B], 0), 1.0 / n)
