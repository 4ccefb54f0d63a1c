"""Polyhedral mesh import: plain-text round trips, a hand-written tetrahedron, and
rejection of invalid files naming the entity (SPEC load_mesh examples)."""
import numpy as np
import pytest

from synthetic import hex_mesh, cvt_mesh
from synthetic.mesh import octa_mesh
from synthetic.meshio import save_mesh, load_mesh, validate

TET = """# vbddc-polymesh 1
vertices 4
0 0 0
1 0 0
0 1 0
0 0 1
faces 4
1 3 0 2 1
1 3 0 1 3
1 3 0 3 2
1 3 1 2 3
cells 1
4 0 1 1 1 2 1 3 1
"""


def _same(a, b):
    for f in ("xyz", "face_ptr", "face_vtx", "cell_ptr", "cell_face", "cell_face_sign", "face_on_boundary"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


@pytest.mark.parametrize("make", [lambda: hex_mesh(2), lambda: hex_mesh(2, jitter=0.2, seed=3, triangulate=True),
                                  lambda: cvt_mesh(3, seed=5), lambda: octa_mesh(2)])
def test_round_trip(tmp_path, make):
    m = make()
    validate(m)
    p = tmp_path / "m.txt"
    save_mesh(m, p)
    _same(m, load_mesh(p))


def test_tetrahedron_file(tmp_path):
    p = tmp_path / "tet.txt"
    p.write_text(TET)
    m = load_mesh(p)
    assert m.n_cells == 1 and m.n_faces == 4 and m.face_on_boundary.all()


def test_rejections_name_the_entity(tmp_path):
    m = hex_mesh(2)
    bad = hex_mesh(2)
    v = bad.face(5)[0]
    bad.xyz = bad.xyz.copy()
    bad.xyz[v] += np.array([1e-3, 1e-3, 1e-3])          # breaks planarity of every face at v
    with pytest.raises(ValueError, match="face .*non-planar"):
        validate(bad)
    open_cell = hex_mesh(2)
    open_cell.cell_face_sign = open_cell.cell_face_sign.copy()
    open_cell.cell_face_sign[0] = -open_cell.cell_face_sign[0]
    with pytest.raises(ValueError, match="cell 0"):
        validate(open_cell)
    p = tmp_path / "t.txt"
    p.write_text(TET.replace("1 3 1 2 3", "1 3 1 2 9"))
    with pytest.raises(ValueError, match="face 3"):
        load_mesh(p)


def test_octa_cells_are_truncated_octahedra():
    """OCTA cells away from the clipped boundary layer are 14-faced truncated octahedra (8 hexagons,
    6 squares; SPEC example n=4); the cell of the lattice point nearest the centre is one of them."""
    m = octa_mesh(4)
    K = int(np.argmin(np.linalg.norm(m.generators - 0.5, axis=1)))
    fs, _ = m.cell_faces(K)
    assert sorted(len(m.face(f)) for f in fs) == [4] * 6 + [6] * 8
    n_to = sum(sorted(len(m.face(f)) for f in m.cell_faces(q)[0]) == [4] * 6 + [6] * 8 for q in range(m.n_cells))
    assert m.n_cells == 128 and n_to >= 8
    validate(m)


@pytest.mark.parametrize("m", [4, 5, 6])
def test_generated_cvt_meshes_validate(m):
    """The CVT meshes of the GPU tests (default seed) pass the importer's checks: planar faces to
    1e-10 h_f (vertices refined onto their bisector planes), closed cells, consistent incidence."""
    from synthetic import make_cvt_problem
    validate(make_cvt_problem(m).mesh)
