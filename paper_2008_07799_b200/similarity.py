"""Similarity types and the K2/K3 kernels (drop-in for drgraph.similarity).

``build_sparse_similarity`` keeps the reference signature and result type
(similarity.py:56-107, 216-278); the per-row perplexity bisection, the
conditional rows and the symmetrisation run in one C-ABI call (drg_similarity).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import DeviceNeighborDistances, NeighborDistances


@dataclass
class SimilarityParams:
    """similarity.py:31-53, plus the BASELINE C3 extension ``neighbor_cap``
    (keep the (dist,id)-sorted prefix of each k-hop row)."""

    k: int = 1
    perplexity: float | str = "auto"
    tol: float = 1e-5
    max_iter: int = 64
    sigma_min: float = 1e-5
    sigma_max: float = 1e5
    neighbor_cap: int | None = None

    def __post_init__(self) -> None:
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if self.k > 6:
            raise ValueError("k > 6 is unsupported (neighborhoods explode)")
        if self.perplexity != "auto" and not self.perplexity >= 1:
            raise ValueError("perplexity must be >= 1 or 'auto'")
        if self.neighbor_cap is not None and self.neighbor_cap < 1:
            raise ValueError("neighbor_cap must be >= 1")


@dataclass(frozen=True)
class SparseSimilarity:
    """Symmetric normalised similarity stored directed (similarity.py:56-107)."""

    indptr: np.ndarray
    targets: np.ndarray
    weights: np.ndarray
    total_mass: float
    sigma: np.ndarray
    k: int

    @property
    def node_count(self) -> int:
        return len(self.indptr) - 1

    @property
    def entry_count(self) -> int:
        return len(self.targets)

    def row(self, i: int):
        lo, hi = self.indptr[i], self.indptr[i + 1]
        return self.targets[lo:hi], self.weights[lo:hi]

    def row_masses(self) -> np.ndarray:
        if self.node_count == 0 or len(self.weights) == 0:
            return np.zeros(self.node_count, dtype=np.float64)
        return np.add.reduceat(np.append(self.weights, 0.0),
                               self.indptr[:-1]) * (np.diff(self.indptr) > 0)

    def sources(self) -> np.ndarray:
        return np.repeat(np.arange(self.node_count, dtype=np.int32), np.diff(self.indptr))

    def nbytes(self) -> int:
        return (self.indptr.nbytes + self.targets.nbytes + self.weights.nbytes
                + self.sigma.nbytes)

    def dump_text(self) -> str:
        src = self.sources()
        lines = [f"{int(i)} {int(j)} {w:.17g}" for i, j, w in zip(src, self.targets, self.weights)]
        return "\n".join(lines) + ("\n" if lines else "")


@dataclass
class DeviceSimilarity:
    """P resident in HBM: CSR (indptr int64, targets int32, weights fp64) plus
    sigma and the per-node incident mass r (the negative-sampler basis)."""

    indptr: torch.Tensor
    targets: torch.Tensor
    weights: torch.Tensor
    sigma: torch.Tensor
    row_mass: torch.Tensor
    total_mass: float
    n_nonisolated: int
    k: int

    @property
    def node_count(self) -> int:
        return self.indptr.numel() - 1

    @property
    def entry_count(self) -> int:
        return self.targets.numel()

    def nbytes(self) -> int:
        return (self.indptr.numel() * 8 + self.targets.numel() * 4 + self.weights.numel() * 8
                + self.sigma.numel() * 8)

    def to_host(self) -> SparseSimilarity:
        return SparseSimilarity(self.indptr.cpu().numpy(), self.targets.cpu().numpy(),
                                self.weights.cpu().numpy(), float(self.total_mass),
                                self.sigma.cpu().numpy(), self.k)


def device_similarity(nd: DeviceNeighborDistances, params: SimilarityParams | None = None
                      ) -> DeviceSimilarity:
    """K2 + K3 on resident k-hop rows (drg_similarity)."""
    params = params or SimilarityParams(k=nd.k)
    if nd.cap:
        return device_similarity_union(nd, params)
    n, nnz = nd.node_count, nd.nnz
    dev = nd.indptr.device
    sigma = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    weights = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    row_mass = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    total = _lib.out_f64()
    n_ne = _lib.out_i64()
    perp = -1.0 if params.perplexity == "auto" else float(params.perplexity)
    _lib.call("drg_similarity", _lib.ptr(nd.indptr), _lib.ptr(nd.ids), _lib.ptr(nd.dists), n,
              nnz, nd.k, perp, float(params.tol), int(params.max_iter), float(params.sigma_min),
              float(params.sigma_max), _lib.ptr(sigma), _lib.ptr(weights), _lib.ptr(row_mass),
              _lib.byref(total), _lib.byref(n_ne), _lib.stream_ptr())
    return DeviceSimilarity(nd.indptr, nd.ids, weights[:nnz], sigma[:n], row_mass[:n],
                            total.value, n_ne.value, nd.k)


def device_similarity_union(nd: DeviceNeighborDistances, params: SimilarityParams
                            ) -> DeviceSimilarity:
    """Capped rows (BASELINE C3): conditional rows over the capped prefixes, then
    union symmetrisation (drg_similarity_union); rows of the result are id-sorted."""
    n, nnz = nd.node_count, nd.nnz
    dev = nd.indptr.device
    sigma = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    indptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    targets = torch.empty(max(2 * nnz, 1), dtype=torch.int32, device=dev)
    weights = torch.empty(max(2 * nnz, 1), dtype=torch.float64, device=dev)
    row_mass = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    out_nnz, total, n_ne = _lib.out_i64(), _lib.out_f64(), _lib.out_i64()
    perp = -1.0 if params.perplexity == "auto" else float(params.perplexity)
    _lib.call("drg_similarity_union", _lib.ptr(nd.indptr), _lib.ptr(nd.ids), _lib.ptr(nd.dists),
              n, nnz, nd.k, perp, float(params.tol), int(params.max_iter),
              float(params.sigma_min), float(params.sigma_max), _lib.ptr(sigma), _lib.ptr(indptr),
              _lib.ptr(targets), _lib.ptr(weights), _lib.ptr(row_mass), _lib.byref(out_nnz),
              _lib.byref(total), _lib.byref(n_ne), _lib.stream_ptr())
    m = out_nnz.value
    return DeviceSimilarity(indptr, targets[:m].clone(), weights[:m].clone(), sigma[:n],
                            row_mass[:n], total.value, n_ne.value, nd.k)


def build_sparse_similarity(nd: NeighborDistances,
                            params: SimilarityParams | None = None) -> SparseSimilarity:
    """similarity.py:216-278 on the GPU.  P matches the reference within 1e-12
    relative (fp64 throughout; exp/log2 may differ by an ulp), stored entries are
    bitwise symmetric, and ``total_mass`` is the device sum of the weights."""
    if params is None:
        params = SimilarityParams()
    _lib.load()
    dnd = DeviceNeighborDistances.from_host(nd)
    if params.neighbor_cap:
        dnd.cap = int(params.neighbor_cap)
    ds = device_similarity(dnd, params)
    return ds.to_host()


# ---------------------------------------------------------------------------
# single-row helpers of the reference API, on the device (rowops.cu)
# ---------------------------------------------------------------------------

def _row_tensors(row) -> tuple[torch.Tensor, torch.Tensor]:
    d = np.fromiter((int(dd) for _, dd in row), dtype=np.int32, count=len(row))
    indptr = torch.tensor([0, len(d)], dtype=torch.int64, device="cuda")
    return indptr, torch.from_numpy(d).cuda()


def precompute_gaussian_table(k: int, sigma: float) -> np.ndarray:
    """Gaussian kernel values exp(-d^2 / (2 sigma^2)) for the hop distances 1..k
    (similarity.py:110-119), by drg_gaussian_table."""
    if k < 1:
        raise ValueError("k must be >= 1")
    _lib.load()
    out = torch.empty(k, dtype=torch.float64, device="cuda")
    _lib.call("drg_gaussian_table", int(k), float(sigma), _lib.ptr(out), _lib.stream_ptr())
    return out.cpu().numpy()


def conditional_similarity_row(row, sigma: float) -> list[tuple[int, float]]:
    """Gaussian conditional probabilities of one node's (neighbour id, hop distance)
    pairs (similarity.py:122-145): p = table[d] / fsum(row); [] for an empty row;
    uniform over the nearest entries if every kernel value underflows
    (drg_rows_conditional)."""
    row = list(row)
    if not row:
        return []
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    _lib.load()
    indptr, dists = _row_tensors(row)
    sig = torch.tensor([float(sigma)], dtype=torch.float64, device="cuda")
    p = torch.empty(len(row), dtype=torch.float64, device="cuda")
    _lib.call("drg_rows_conditional", _lib.ptr(indptr), _lib.ptr(dists), 1, _lib.ptr(sig),
              _lib.ptr(p), _lib.stream_ptr())
    return [(int(j), float(v)) for (j, _), v in zip(row, p.cpu().tolist())]


def search_sigma(row, perplexity: float, tol: float = 1e-5, max_iter: int = 64,
                 sigma_min: float = 1e-5, sigma_max: float = 1e5) -> float:
    """Geometric bisection for the bandwidth whose row perplexity matches the target
    clamped to [1, len(row)] (similarity.py:167-199), by drg_rows_sigma -- the same
    device routine build_sparse_similarity's rows use."""
    row = list(row)
    if not row:
        raise ValueError("cannot search sigma for an empty row")
    if len(row) == 1:
        return 1.0
    _lib.load()
    indptr, dists = _row_tensors(row)
    out = torch.ones(1, dtype=torch.float64, device="cuda")
    _lib.call("drg_rows_sigma", _lib.ptr(indptr), _lib.ptr(dists), 1, float(perplexity),
              float(tol), int(max_iter), float(sigma_min), float(sigma_max), _lib.ptr(out),
              _lib.stream_ptr())
    return float(out.item())

