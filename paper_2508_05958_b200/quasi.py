"""Quasi-uniform triangle-mesh pipeline on the B200 (drop-in for ``htlr.quasi``,
/root/reference/pkg/src/htlr/quasi.py).

Centroid values are moved to an auxiliary uniform grid by the area-overlap
matrix S, multiplied by the HTLR operator there, and moved back by the
reverse-overlap matrix T.  The mesh container and file I/O are host objects
as in the reference; the overlap areas (Sutherland-Hodgman clipping) and
both sparse transfers run on the device (``htlr_overlap_areas``,
``htlr_csr_spmv``); the CSR assembly uses torch device sorts.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .grids import UniformGrid, leaf_side_for
from .operators import BuildConfig, HTLRMatrix, construct, matvec

COVERAGE_TOL = 1e-8   # quasi.py:20


@dataclass
class TriMesh:
    """Triangulation of [0,1]^2 (quasi.py:23-59)."""

    vertices: np.ndarray
    triangles: np.ndarray
    centroids: np.ndarray = field(init=False)
    areas: np.ndarray = field(init=False)

    def __post_init__(self):
        self.vertices = np.asarray(self.vertices, dtype=np.float64)
        self.triangles = np.asarray(self.triangles, dtype=np.int64)
        if self.triangles.size and (self.triangles.min() < 0 or self.triangles.max() >= len(self.vertices)):
            raise ValueError("triangle vertex index out of range")
        c = self.vertices[self.triangles]
        self.centroids = c.mean(axis=1)
        e1 = c[:, 1] - c[:, 0]
        e2 = c[:, 2] - c[:, 0]
        self.areas = 0.5 * np.abs(e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0])
        if np.any(self.areas <= 0.0):
            raise ValueError("mesh contains a zero-area triangle")
        gap = abs(float(self.areas.sum()) - 1.0)
        if gap > COVERAGE_TOL:
            raise ValueError(f"mesh does not cover the unit square (area deficit {gap:.2e})")

    @property
    def num_triangles(self) -> int:
        return len(self.triangles)

    def corners(self, i: int) -> np.ndarray:
        return self.vertices[self.triangles[i]]


def load_mesh(path) -> TriMesh:
    """'V F' header, V lines 'x y', F lines of 1-based 'i j k' (quasi.py:62-83)."""
    with open(path) as fh:
        tok = fh.read().split()
    if len(tok) < 2:
        raise ValueError("mesh file too short")
    try:
        nv, nf = int(tok[0]), int(tok[1])
        body = tok[2:]
        if len(body) != 2 * nv + 3 * nf:
            raise ValueError(f"expected {2 * nv + 3 * nf} values after the header, got {len(body)}")
        verts = np.array(body[:2 * nv], dtype=np.float64).reshape(nv, 2)
        tris = np.array(body[2 * nv:], dtype=np.int64).reshape(nf, 3) - 1
    except ValueError:
        raise
    except Exception as exc:
        raise ValueError(f"malformed mesh file: {exc}") from exc
    return TriMesh(vertices=verts, triangles=tris)


def save_mesh(mesh: TriMesh, path) -> None:
    with open(path, "w") as fh:
        fh.write(f"{len(mesh.vertices)} {len(mesh.triangles)}\n")
        fh.writelines(f"{float(x)!r} {float(y)!r}\n" for x, y in mesh.vertices)
        fh.writelines(f"{a + 1} {b + 1} {c + 1}\n" for a, b, c in mesh.triangles)


def structured_trimesh(cells_per_side: int, diagonal: str = "down") -> TriMesh:
    """k x k cells, two triangles each (quasi.py:95-120)."""
    k = cells_per_side
    if k < 1:
        raise ValueError("cells_per_side must be >= 1")
    if diagonal not in ("down", "up"):
        raise ValueError("diagonal must be 'down' or 'up'")
    xs = np.arange(k + 1) / k
    jj, ii = np.meshgrid(np.arange(k + 1), np.arange(k + 1), indexing="ij")
    verts = np.stack([xs[ii.ravel()], xs[jj.ravel()]], axis=-1)

    def vid(i, j):
        return i + j * (k + 1)

    tris = []
    for j in range(k):
        for i in range(k):
            a, b, c, d = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
            tris += [(a, b, d), (b, c, d)] if diagonal == "down" else [(a, b, c), (a, c, d)]
    return TriMesh(vertices=verts, triangles=np.array(tris))


@dataclass
class SparseInterpMatrix:
    """Device CSR transfer matrix (quasi.py:174-195)."""

    indptr: object      # torch int64 (rows + 1), device
    indices: object     # torch int32, device
    data: object        # torch float64, device
    shape: tuple

    @property
    def rows(self) -> int:
        return self.shape[0]

    @property
    def cols(self) -> int:
        return self.shape[1]

    def row_sums(self) -> np.ndarray:
        import torch
        rid = torch.repeat_interleave(torch.arange(self.rows, device=self.data.device),
                                      self.indptr[1:] - self.indptr[:-1])
        s = torch.zeros(self.rows, dtype=torch.float64, device=self.data.device).index_add_(0, rid, self.data)
        return s.cpu().numpy()

    def entries_in_row(self, row: int) -> int:
        return int(self.indptr[row + 1] - self.indptr[row])

    def toarray(self) -> np.ndarray:
        out = np.zeros(self.shape)
        ip = self.indptr.cpu().numpy()
        ix = self.indices.cpu().numpy()
        dv = self.data.cpu().numpy()
        for r in range(self.rows):
            out[r, ix[ip[r]:ip[r + 1]]] += dv[ip[r]:ip[r + 1]]
        return out

    def apply_device(self, x):
        import torch
        y = torch.empty(self.rows, dtype=torch.float64, device=x.device)
        st = torch.cuda.current_stream(x.device).cuda_stream
        _lib.check(_lib.lib().htlr_csr_spmv(ctypes.c_void_p(self.indptr.data_ptr()),
                                            ctypes.c_void_p(self.indices.data_ptr()),
                                            ctypes.c_void_p(self.data.data_ptr()), self.rows,
                                            ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                            ctypes.c_void_p(st)))
        return y

    def apply(self, v: np.ndarray) -> np.ndarray:
        import torch
        x = torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.float64))).to(self.data.device)
        return self.apply_device(x).cpu().numpy()


def _overlap_entries(mesh: TriMesh, m_side: int, device=None):
    """(cell, triangle, area) triples with positive overlap (quasi.py:198-219);
    candidate cells from each triangle's bounding box (host integer work),
    areas on the device."""
    import torch
    if device is None:
        device = torch.cuda.current_device()
    c = mesh.vertices[mesh.triangles]
    lo = c.min(axis=1)
    hi = c.max(axis=1)
    i0 = np.maximum(np.floor(lo[:, 0] * m_side).astype(np.int64), 0)
    i1 = np.minimum(np.ceil(hi[:, 0] * m_side).astype(np.int64), m_side)
    j0 = np.maximum(np.floor(lo[:, 1] * m_side).astype(np.int64), 0)
    j1 = np.minimum(np.ceil(hi[:, 1] * m_side).astype(np.int64), m_side)
    ni = np.maximum(i1 - i0, 0)
    nj = np.maximum(j1 - j0, 0)
    cnt = ni * nj
    tri = np.repeat(np.arange(mesh.num_triangles), cnt)
    off = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    ci = i0[tri] + off % ni[tri]
    cj = j0[tri] + off // ni[tri]
    cand = np.ascontiguousarray(np.stack([tri, ci, cj], axis=-1).astype(np.int32))
    dev = torch.device("cuda", device)
    txy = torch.from_numpy(np.ascontiguousarray(c.reshape(-1, 6))).to(dev)
    dcand = torch.from_numpy(cand).to(dev)
    areas = torch.empty(len(cand), dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.lib().htlr_overlap_areas(ctypes.c_void_p(txy.data_ptr()), ctypes.c_void_p(dcand.data_ptr()),
                                             len(cand), m_side, ctypes.c_void_p(areas.data_ptr()),
                                             ctypes.c_void_p(st)))
    h = 1.0 / m_side
    keep = areas > 1e-13 * (h * h)
    cells = (dcand[:, 1].long() + dcand[:, 2].long() * m_side)[keep]
    return cells, dcand[:, 0].long()[keep], areas[keep]


def _csr(rows, cols, vals, shape) -> SparseInterpMatrix:
    import torch
    key = rows * shape[1] + cols
    order = torch.argsort(key)
    rows, cols, vals = rows[order], cols[order], vals[order]
    counts = torch.bincount(rows, minlength=shape[0])
    indptr = torch.zeros(shape[0] + 1, dtype=torch.int64, device=vals.device)
    indptr[1:] = torch.cumsum(counts, 0)
    return SparseInterpMatrix(indptr=indptr, indices=cols.to(torch.int32).contiguous(),
                              data=vals.contiguous(), shape=shape)


def quasi_to_uniform(mesh: TriMesh, m_side: int) -> SparseInterpMatrix:
    """S (M x N): overlap of cell t with triangle i over the cell area (quasi.py:222-243)."""
    cells, tris, areas = _overlap_entries(mesh, m_side)
    mat = _csr(cells, tris, areas * (m_side * m_side), (m_side * m_side, mesh.num_triangles))
    bad = np.abs(mat.row_sums() - 1.0) > COVERAGE_TOL
    if np.any(bad):
        raise ValueError(f"{int(bad.sum())} uniform cells are not fully covered by the mesh")
    return mat


def uniform_to_quasi(mesh: TriMesh, m_side: int) -> SparseInterpMatrix:
    """T (N x M): overlap of triangle i with cell t over the triangle area (quasi.py:246-261)."""
    import torch
    cells, tris, areas = _overlap_entries(mesh, m_side)
    tri_area = torch.from_numpy(mesh.areas).to(areas.device)
    mat = _csr(tris, cells, areas / tri_area[tris], (mesh.num_triangles, m_side * m_side))
    bad = np.abs(mat.row_sums() - 1.0) > COVERAGE_TOL
    if np.any(bad):
        raise ValueError(f"{int(bad.sum())} triangles stick out of the uniform grid")
    return mat


@dataclass
class QuasiPipeline:
    to_quasi: SparseInterpMatrix
    op: HTLRMatrix
    to_uniform: SparseInterpMatrix
    m_side: int
    rho: float


def valid_uniform_side(target: int, leaf_side: int) -> int:
    """Nearest side to `target` that halves evenly to the leaf (quasi.py:264-277)."""
    for delta in range(max(target, 4)):
        for cand in (target + delta, target - delta):
            if cand < 1:
                continue
            try:
                leaf_side_for(cand, leaf_side)
            except ValueError:
                continue
            return cand
    raise ValueError("no valid uniform grid side near the target")


def build_pipeline(mesh: TriMesh, cfg: BuildConfig, rho: float, threads: int = 1) -> QuasiPipeline:
    """quasi.py:280-300."""
    target = int(round(np.sqrt(rho * rho * mesh.num_triangles / 2.0)))
    m_side = valid_uniform_side(max(target, cfg.leaf_side), cfg.leaf_side)
    op = construct(cfg, UniformGrid(2, m_side))
    s_mat = quasi_to_uniform(mesh, m_side)
    t_mat = uniform_to_quasi(mesh, m_side)
    return QuasiPipeline(to_quasi=t_mat, op=op, to_uniform=s_mat, m_side=m_side,
                         rho=float(np.sqrt(2.0 * m_side * m_side / mesh.num_triangles)))


def apply_pipeline(pipe: QuasiPipeline, u):
    """T (A (S u)) on the device (quasi.py:303-313); numpy in -> numpy out."""
    import torch
    host = not (isinstance(u, torch.Tensor) and u.is_cuda)
    x = u if isinstance(u, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(u, dtype=np.float64)))
    x = x.reshape(-1)
    if x.numel() != pipe.to_uniform.cols:
        raise ValueError("vector length does not match the mesh")
    x = x.to(pipe.to_uniform.data.device, dtype=torch.float64)
    y = pipe.to_quasi.apply_device(matvec(pipe.op, pipe.to_uniform.apply_device(x)))
    return y.cpu().numpy() if host else y


def overlap_area(tri, cell) -> float:
    """Area of triangle intersect rectangle (x0, y0, x1, y1) (quasi.py:152-171),
    computed by the device clipping kernel: the cell is placed as cell (0, 0)
    of a unit grid after an affine map of the triangle."""
    import torch
    x0, y0, x1, y1 = cell
    tri = np.asarray(tri, dtype=np.float64)
    # map the rectangle to the unit cell [0, 1]^2 of a 1x1 grid
    sx, sy = x1 - x0, y1 - y0
    t = np.stack([(tri[:, 0] - x0) / sx, (tri[:, 1] - y0) / sy], axis=-1).reshape(1, 6)
    dev = torch.device("cuda", torch.cuda.current_device())
    txy = torch.from_numpy(np.ascontiguousarray(t)).to(dev)
    cand = torch.zeros(3, dtype=torch.int32, device=dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.lib().htlr_overlap_areas(ctypes.c_void_p(txy.data_ptr()), ctypes.c_void_p(cand.data_ptr()), 1,
                                             1, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st)))
    return float(out.item()) * sx * sy
