"""Plain-text polyhedral mesh files (SPEC's "documented plain-text polyhedral format":
counts header, vertex coordinates, faces as vertex loops, cells as signed face lists), so meshes
produced elsewhere (CVT, OCTA, agglomerates) can be imported.  Input plumbing only: validation
is geometric bookkeeping (planarity, closedness, face incidence), none of the method's arithmetic.

    # vbddc-polymesh 1
    vertices <nV>
    <x> <y> <z>                          (nV lines)
    faces <nF>
    <boundary 0|1> <len> <v_0> ... <v_len-1>   (nF lines, loop order = orientation)
    cells <nK>
    <nf> <f_0> <s_0> ... <f_nf-1> <s_nf-1>     (nK lines, s = +1 iff the loop normal points out)
"""
import numpy as np

from .mesh import PolyMesh

HEADER = "# vbddc-polymesh 1"


def save_mesh(mesh, path):
    with open(path, "w") as f:
        f.write(HEADER + "\n")
        f.write("vertices %d\n" % mesh.n_vertices)
        for x in mesh.xyz:
            f.write("%.17g %.17g %.17g\n" % tuple(x))
        f.write("faces %d\n" % mesh.n_faces)
        for i in range(mesh.n_faces):
            lp = mesh.face(i)
            f.write("%d %d %s\n" % (int(mesh.face_on_boundary[i]), len(lp), " ".join(str(int(v)) for v in lp)))
        f.write("cells %d\n" % mesh.n_cells)
        for K in range(mesh.n_cells):
            fs, ss = mesh.cell_faces(K)
            f.write("%d %s\n" % (len(fs), " ".join("%d %d" % (int(a), int(b)) for a, b in zip(fs, ss))))


def _face_frame(X):
    """Newell normal (area vector / 2) and diameter of a polygon loop X [n,3]."""
    a = np.zeros(3)
    for i in range(len(X)):
        a += np.cross(X[i], X[(i + 1) % len(X)])
    a *= 0.5
    diam = max(np.linalg.norm(X[i] - X[j]) for i in range(len(X)) for j in range(i + 1, len(X)))
    return a, diam


def validate(mesh, planar_tol=1e-10, closed_tol=1e-12):
    """Reject a mesh that is not a valid polyhedral partition, naming the entity: a face with fewer than
    3 vertices or non-planar beyond planar_tol * h_f; a cell whose boundary is open
    (|sum_f s_f area_f n_f| > closed_tol h_K^2) or has non-positive volume; a face used by more than
    two cells, by two cells with equal signs, or flagged inconsistently as boundary."""
    nF, nK = mesh.n_faces, mesh.n_cells
    areavec = np.zeros((nF, 3))
    for f in range(nF):
        lp = mesh.face(f)
        if len(lp) < 3 or len(set(lp.tolist())) != len(lp):
            raise ValueError("face %d: degenerate vertex loop" % f)
        X = mesh.xyz[lp]
        a, diam = _face_frame(X)
        nrm = a / np.linalg.norm(a)
        dev = np.abs((X - X.mean(0)) @ nrm).max()
        if dev > planar_tol * diam:
            raise ValueError("face %d: non-planar (%.2e > %.1e h_f)" % (f, dev / diam, planar_tol))
        areavec[f] = a
    use = [[] for _ in range(nF)]
    for K in range(nK):
        fs, ss = mesh.cell_faces(K)
        acc = np.zeros(3)
        vol = 0.0
        verts = np.unique(np.concatenate([mesh.face(f) for f in fs]))
        hK = max(np.linalg.norm(mesh.xyz[verts] - x, axis=1).max() for x in mesh.xyz[verts])
        for f, s in zip(fs, ss):
            if s not in (1, -1):
                raise ValueError("cell %d: face sign %d is not +-1" % (K, s))
            acc += s * areavec[f]
            vol += s * areavec[f] @ mesh.xyz[mesh.face(f)].mean(0) / 3.0
            use[f].append((K, s))
        if np.linalg.norm(acc) > closed_tol * hK * hK:
            raise ValueError("cell %d: open boundary (|sum s_f a_f| = %.2e h_K^2)" % (K, np.linalg.norm(acc) / hK ** 2))
        if vol <= 0:
            raise ValueError("cell %d: non-positive volume %.3e (face signs)" % (K, vol))
    for f in range(nF):
        u = use[f]
        if len(u) == 0 or len(u) > 2:
            raise ValueError("face %d: used by %d cells" % (f, len(u)))
        if len(u) == 2 and u[0][1] == u[1][1]:
            raise ValueError("face %d: equal orientation in cells %d and %d" % (f, u[0][0], u[1][0]))
        if (len(u) == 1) != bool(mesh.face_on_boundary[f]):
            raise ValueError("face %d: boundary flag inconsistent with its %d cell(s)" % (f, len(u)))
    return mesh


def load_mesh(path, h=None):
    """Read and validate a mesh file (ValueError naming the line or entity on failure)."""
    with open(path) as fh:
        lines = [l.strip() for l in fh if l.strip() and not l.startswith("#")]
    it = iter(lines)

    def section(name):
        head = next(it).split()
        if head[0] != name or len(head) != 2:
            raise ValueError("expected '%s <count>', got %r" % (name, " ".join(head)))
        return int(head[1])

    nV = section("vertices")
    xyz = np.array([[float(t) for t in next(it).split()] for _ in range(nV)], dtype=np.float64).reshape(nV, 3)
    nF = section("faces")
    fb, ptr, vtx = [], [0], []
    for f in range(nF):
        t = [int(x) for x in next(it).split()]
        if len(t) != 2 + t[1]:
            raise ValueError("face %d: loop length %d does not match its %d entries" % (f, t[1], len(t) - 2))
        if min(t[2:]) < 0 or max(t[2:]) >= nV:
            raise ValueError("face %d: vertex id out of range" % f)
        fb.append(t[0]); vtx += t[2:]; ptr.append(len(vtx))
    nK = section("cells")
    cptr, cf, cs = [0], [], []
    for K in range(nK):
        t = [int(x) for x in next(it).split()]
        if len(t) != 1 + 2 * t[0]:
            raise ValueError("cell %d: face count %d does not match its entries" % (K, t[0]))
        if min(t[1::2]) < 0 or max(t[1::2]) >= nF:
            raise ValueError("cell %d: face id out of range" % K)
        cf += t[1::2]; cs += t[2::2]; cptr.append(len(cf))
    mesh = PolyMesh(xyz, np.array(ptr, dtype=np.int64), np.array(vtx, dtype=np.int64), np.array(cptr, dtype=np.int64),
                    np.array(cf, dtype=np.int64), np.array(cs, dtype=np.int8), np.array(fb, dtype=np.uint8), None,
                    (0, 0, 0), h if h is not None else nK ** (-1.0 / 3.0))
    return validate(mesh)
