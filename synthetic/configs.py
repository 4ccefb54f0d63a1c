"""The five BASELINE.json configurations as seeded synthetic inputs.

Each config yields a `Problem`: the mesh, the box partition, the per-cell
viscosity array and the parameters of the analytic data.  The analytic fields
(manufactured u, p, f and the sinker force) are *named* here with their
parameters; each side (oracle, CUDA library) evaluates them with its own code.

Manufactured (configs 1,2,3,5; BASELINE.json configs[0,1,2,4]):
    psi = sin(pi x) sin(pi y) sin(pi z) (1,1,1),  u = curl psi,
    p = sin(2 pi x) cos(pi y) z  (its mean over [0,1]^3 is 0),
    f = -div(nu eps(u)) - grad p = (3 pi^2 nu / 2) u - grad p.
Multi-sinker (config 4; BASELINE.json configs[3]):
    chi(x) = prod_i [1 - exp(-delta max(0, |x-c_i| - omega/2)^2)],
    nu(x) = (nu_max - nu_min)(1 - chi) + nu_min, f = (0, 0, beta (chi - 1)),
    c_i = default_rng(seed).uniform(0.1, 0.9, (8, 3)); nu_K = nu(vertex mean of K).
"""
from dataclasses import dataclass, field
import numpy as np
from .mesh import hex_mesh, box_partition, cvt_mesh, centroid_partition, octa_mesh, mark_neumann


@dataclass
class Problem:
    name: str
    k: int
    mesh: object
    cell_subdomain: np.ndarray
    sub_grid: tuple
    nu_cell: np.ndarray
    kind: str                      # "manufactured" | "sinker"
    constraints: dict = field(default_factory=dict)
    rtol: float = 1e-10
    params: dict = field(default_factory=dict)


SINKER = dict(nu_min=1e-2, nu_max=1e2, delta=200.0, omega=0.1, beta=10.0, n_sinkers=8)


def sinker_centres(seed):
    return np.random.default_rng(seed).uniform(0.1, 0.9, (SINKER["n_sinkers"], 3))


def sinker_chi(x, centres):
    """chi(x) for points x [...,3] (input recipe only: used for the viscosity array)."""
    chi = np.ones(x.shape[:-1])
    for c in centres:
        d = np.linalg.norm(x - c, axis=-1)
        chi *= 1.0 - np.exp(-SINKER["delta"] * np.maximum(0.0, d - SINKER["omega"] / 2) ** 2)
    return chi


def _cell_vertex_mean(mesh):
    nK = mesh.n_cells
    out = np.zeros((nK, 3))
    for K in range(nK):
        fs, _ = mesh.cell_faces(K)
        vs = np.unique(np.concatenate([mesh.face(f) for f in fs]))
        out[K] = mesh.xyz[vs].mean(0)
    return out


def _cell_vertex_mean_structured(mesh):
    h = mesh.h
    return (mesh.cell_ijk + 0.5) * h


CONFIGS = {
    # name: (n, dims, sub, k, jitter, triangulate, kind, constraints)
    "c1": dict(n=4, dims=None, sub=(2, 2, 2), k=2, jitter=0.0, tri=False, kind="manufactured",
               constraints=dict(vertex=1, edge_avg=1, face_avg=1, face_flux=1, adaptive_tau=0.0)),
    "c2": dict(n=16, dims=None, sub=(4, 4, 4), k=2, jitter=0.0, tri=False, kind="manufactured",
               constraints=dict(vertex=1, edge_avg=1, face_avg=1, face_flux=1, adaptive_tau=0.0)),
    "c3": dict(n=16, dims=None, sub=(4, 4, 4), k=3, jitter=0.2, tri=True, kind="manufactured",
               constraints=dict(vertex=1, edge_avg=1, face_avg=1, face_flux=1, adaptive_tau=0.0)),
    "c4": dict(n=32, dims=None, sub=(4, 4, 4), k=2, jitter=0.0, tri=False, kind="sinker",
               constraints=dict(vertex=1, edge_avg=1, face_avg=0, face_flux=1, adaptive_tau=10.0)),
    # config 5: per-GPU box of 8^3 subdomains of 4^3 cells, h = 1/32 fixed (weak scaling)
    "c5": dict(n=32, dims=(32, 32, 32), sub=(4, 4, 4), k=2, jitter=0.0, tri=False, kind="manufactured",
               constraints=dict(vertex=1, edge_avg=1, face_avg=1, face_flux=1, adaptive_tau=0.0)),
}

C5_DIMS = {1: (32, 32, 32), 2: (32, 32, 64), 4: (32, 64, 64), 8: (64, 64, 64)}


def make_problem(name, seed=20230419, n=None, sub=None, k=None, dims=None, nu=1.0, kind=None,
                 constraints=None, neumann=None):
    """Build the seeded inputs of config `name`; keyword overrides give small variants.
    neumann: sides of the cube posed with the natural (homogeneous traction) condition, e.g.
    ("x1", "y1") for the paper's two Neumann faces (DESIGN A35)."""
    cfg = dict(CONFIGS[name])
    if n is not None:
        cfg["n"] = n
        if dims is None:
            cfg["dims"] = None
    if dims is not None:
        cfg["dims"] = dims
    if sub is not None:
        cfg["sub"] = sub
    if k is not None:
        cfg["k"] = k
    if kind is not None:
        cfg["kind"] = kind
    cons = dict(cfg["constraints"])
    if constraints is not None:
        cons.update(constraints)
    mesh = hex_mesh(cfg["n"], dims=cfg["dims"], jitter=cfg["jitter"], seed=seed, triangulate=cfg["tri"])
    if neumann:
        mesh = mark_neumann(mesh, neumann)
    cell_sub, grid = box_partition(mesh, cfg["sub"])
    params = {}
    if cfg["kind"] == "sinker":
        centres = sinker_centres(seed)
        chi = sinker_chi(_cell_vertex_mean_structured(mesh), centres)
        nu_cell = (SINKER["nu_max"] - SINKER["nu_min"]) * (1.0 - chi) + SINKER["nu_min"]
        params = dict(SINKER, centres=centres)
    else:
        nu_cell = np.full(mesh.n_cells, float(nu))
        params = dict(nu=float(nu))
    return Problem(name=name, k=cfg["k"], mesh=mesh, cell_subdomain=cell_sub, sub_grid=grid,
                   nu_cell=nu_cell.astype(np.float64), kind=cfg["kind"], constraints=cons,
                   params=params)


def make_cvt_problem(m=5, grid=(2, 2, 2), k=2, seed=20230419, lloyd=20, nu=1.0, constraints=None):
    """The paper's CVT mesh family (Test 3 uses 125 cells): m^3 centroidal Voronoi
    cells of [0,1]^3 (synthetic.mesh.cvt_mesh), box partition into `grid` subdomains by cell
    generator, the manufactured solution of configs 1/2/3/5, vertex + edge + face constraints with
    deluxe scaling, homogeneous Dirichlet data lifted."""
    mesh = cvt_mesh(m, seed=seed, lloyd=lloyd)
    return poly_problem(mesh, grid, k, nu, constraints, name="cvt")


def make_octa_problem(n=3, grid=(2, 2, 2), k=2, nu=1.0, constraints=None):
    """The paper's OCTA family (SPEC reading: clipped BCC truncated-octahedron tiling,
    2 n^3 cells), partitioned and posed like make_cvt_problem."""
    return poly_problem(octa_mesh(n), grid, k, nu, constraints, name="octa")


def poly_problem(mesh, grid=(2, 2, 2), k=2, nu=1.0, constraints=None, name="poly"):
    """A general polyhedral mesh of [0,1]^3 with generators (cvt_mesh, octa_mesh, or an imported mesh
    given `generators` = cell centroids) posed as configs 1/2/3/5: manufactured solution,
    vertex + edge + face constraints, deluxe scaling, box partition into `grid` by generator."""
    cell_sub, g = centroid_partition(mesh, grid)
    cons = dict(vertex=1, edge_avg=1, face_avg=1, face_flux=1, adaptive_tau=0.0)
    if constraints:
        cons.update(constraints)
    return Problem(name=name, k=k, mesh=mesh, cell_subdomain=cell_sub, sub_grid=g,
                   nu_cell=np.full(mesh.n_cells, float(nu)), kind="manufactured", constraints=cons,
                   params=dict(nu=float(nu)))
