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


def box_partition(mesh, sub):
    """Subdomain id per cell for a box partition with `sub`=(sx,sy,sz) cells per subdomain.

    Subdomains are numbered lexicographically (x fastest) over the subdomain grid.
    """
    sx, sy, sz = sub
    nx, ny, nz = mesh.dims
    gx, gy, gz = nx // sx, ny // sy, nz // sz
    c = mesh.cell_ijk
    return ((c[:, 0] // sx) + gx * ((c[:, 1] // sy) + gy * (c[:, 2] // sz))).astype(np.int32), (gx, gy, gz)
