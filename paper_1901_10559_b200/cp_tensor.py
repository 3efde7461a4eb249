"""CP tensors and TensorSketch rank reduction on B200.

Drop-in for the hot-path part of reference ``pkg/src/idsketch/cp_tensor.py``:
``CpTensor`` (:41-128, the input/output container), ``TensorIdResult``
(:200-212), ``tensor_id_from_sketch`` (:235-239), ``check_tensor_id_args``
(:242-263) and ``tensorsketch_id`` (:266-276).  The sketch and the ID run on
the device; the recombined weights ``weights[cols] * coeffs.sum(axis=1)``
(:216) are formed on the host from the returned coefficients so they equal
numpy's own evaluation bit for bit (the reference test
test_cp_tensor.py:193-203 demands array_equal).
"""

import threading
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .linalg import DEFAULT_RANK_TOL
from .matrix_id import DEFAULT_OVERSAMPLE, device_matrix_id, matrix_id
from .sketch import TensorSketchOp

TENSOR_METHODS = ("tensorsketch",)
_MAX_DENSE_ENTRIES = 50_000_000


def _is_cuda(f):
    import torch

    return isinstance(f, torch.Tensor) and f.device.type == "cuda"


def _fortran_cuda(t):
    """CUDA float64 I x R tensor in column-major layout (a view of an
    (R, I) contiguous tensor), the layout the TensorSketch kernel reads."""
    import torch

    t = t.to(torch.float64)
    return t if t.t().is_contiguous() else t.t().contiguous().t()


def _canon_factor(f, n):
    if _is_cuda(f):  # device-resident factor (B200 extension): stays in HBM
        import torch

        if f.dim() != 2:
            raise ValueError(f"factor {n} must be 2-D, got ndim={f.dim()}")
        if f.numel() == 0:
            raise ValueError(f"factor {n} must be nonempty")
        out = _fortran_cuda(f)
        if not bool(torch.isfinite(out).all()):
            raise ValueError(f"factor {n} contains non-finite entries")
        return out
    if sp.issparse(f):
        out = sp.csc_array(f, dtype=np.float64)
        out.sum_duplicates()
        out.eliminate_zeros()
        out.sort_indices()
        if out.nnz and not np.isfinite(out.data).all():
            raise ValueError("a contains non-finite entries")
        return out
    out = np.asfortranarray(f, dtype=np.float64)
    if out.ndim != 2:
        raise ValueError(f"factor {n} must be 2-D, got ndim={out.ndim}")
    if out.size == 0:
        raise ValueError(f"factor {n} must be nonempty")
    if not np.isfinite(out).all():
        raise ValueError(f"factor {n} contains non-finite entries")
    return out


def _col_norms(f):
    if _is_cuda(f):
        import torch

        return torch.linalg.vector_norm(f, dim=0).cpu().numpy()
    if sp.issparse(f):
        return np.sqrt(np.asarray(f.power(2).sum(axis=0)).ravel())
    return np.linalg.norm(f, axis=0)


def _scaled(f, scale):
    if _is_cuda(f):
        import torch

        return _fortran_cuda(f * torch.from_numpy(np.asarray(scale, np.float64)).to(f.device))
    if sp.issparse(f):
        out = sp.csc_array(f @ sp.diags_array(scale), dtype=np.float64)
        out.sum_duplicates()
        out.eliminate_zeros()
        out.sort_indices()
        return out
    return f * scale


def _unit_columns(f, cols):
    """Replace zero columns by e_0 (cp_tensor.py:131-141)."""
    if _is_cuda(f):
        f = f.clone()
        f[:, cols] = 0.0
        f[0, cols] = 1.0
        return _fortran_cuda(f)
    if sp.issparse(f):
        lil = f.tolil()
        for c in cols:
            lil[:, c] = 0.0
            lil[0, c] = 1.0
        return _canon_factor(lil, 0)
    f = f.copy()
    f[:, cols] = 0.0
    f[0, cols] = 1.0
    return f


class CpTensor:
    """CP tensor: nonnegative `weights` (R) and one unit-column factor per mode
    (cp_tensor.py:41-95).  Factors may be numpy, scipy sparse, or (B200
    extension) CUDA tensors, which are normalized on the device and stay in
    HBM: tensorsketch_id then reads them without a host round trip.  Norms and the sign that keeps weights nonnegative
    (applied to mode 0) are folded into the weights; zero columns get weight 0
    and an arbitrary unit vector.  Columns already unit to 1e-12 are kept bit
    for bit, so selecting terms is an exact column-subset operation."""

    def __init__(self, weights, factors):
        if len(factors) == 0:
            raise ValueError("need at least one factor matrix")
        factors = [_canon_factor(f, n) for n, f in enumerate(factors)]
        rank = factors[0].shape[1]
        for n, f in enumerate(factors):
            if f.shape[1] != rank:
                raise ValueError(f"factor {n} has {f.shape[1]} columns, expected {rank}")
        weights = np.asarray(weights, dtype=np.float64).copy()
        if weights.shape != (rank,):
            raise ValueError(f"weights must have length {rank}")
        if not np.isfinite(weights).all():
            raise ValueError("weights must be finite")
        zero_cols = np.zeros(rank, dtype=bool)
        normalized = []
        for f in factors:
            norms = _col_norms(f)
            zero = norms == 0.0
            zero_cols |= zero
            norms = np.where(np.abs(norms - 1.0) <= 1e-12, 1.0, norms)
            if np.any(norms != 1.0):
                f = _scaled(f, 1.0 / np.where(zero, 1.0, norms))
            if zero.any():
                f = _unit_columns(f, np.flatnonzero(zero))
            weights *= np.where(zero, 0.0, norms)
            normalized.append(f)
        negative = weights < 0.0
        if negative.any():
            normalized[0] = _scaled(normalized[0], np.where(negative, -1.0, 1.0))
            weights = np.abs(weights)
        self.weights = weights
        self.factors = normalized
        self.zero_columns = np.flatnonzero(zero_cols)

    @property
    def rank(self):
        return self.weights.size

    @property
    def ndim(self):
        return len(self.factors)

    @property
    def mode_dims(self):
        return tuple(f.shape[0] for f in self.factors)

    @property
    def total_entries(self):
        return int(np.prod(self.mode_dims))

    def select(self, cols, weights):
        """CP tensor built from the given term indices and new weights."""
        if all(isinstance(f, np.ndarray) for f in self.factors):
            return self._select_dense(cols, weights)
        sel = []
        for f in self.factors:
            if _is_cuda(f):
                import torch

                sel.append(f[:, torch.as_tensor(np.asarray(cols, np.int64), device=f.device)])
            else:
                sel.append(f[:, cols])
        return CpTensor(weights, sel)

    def _select_dense(self, cols, weights):
        """select() for dense host factors without re-validating them: the
        chosen columns are already unit to 1e-12 (this tensor's own
        normalization), so CpTensor(weights, sel) would keep them bit for bit
        and only move negative weights' signs into mode 0 -- which is all
        this does."""
        cols = np.asarray(cols, dtype=np.int64)
        weights = np.asarray(weights, dtype=np.float64).copy()
        if weights.shape != (cols.size,):
            raise ValueError(f"weights must have length {cols.size}")
        if not np.isfinite(weights).all():
            raise ValueError("weights must be finite")
        sel = [np.asfortranarray(f[:, cols]) for f in self.factors]
        negative = weights < 0.0
        if negative.any():
            sel[0] = sel[0] * np.where(negative, -1.0, 1.0)
            weights = np.abs(weights)
        out = object.__new__(CpTensor)
        out.weights = weights
        out.factors = sel
        out.zero_columns = np.zeros(0, dtype=np.int64)
        return out

    def to_dense(self, max_entries=_MAX_DENSE_ENTRIES):
        """Materialize the full tensor (testing and small problems only)."""
        if self.total_entries > max_entries:
            raise ValueError("tensor too large to densify")
        out = np.zeros(self.mode_dims)
        host = [f.cpu().numpy() if _is_cuda(f) else f for f in self.factors]
        for r in range(self.rank):
            term = np.array(self.weights[r])
            for f in host:
                col = f[:, [r]].toarray().ravel() if sp.issparse(f) else f[:, r]
                term = np.multiply.outer(term, col)
            out += term
        return out


@dataclass(frozen=True)
class TensorIdResult:
    """Rank reduction output (cp_tensor.py:200-212): new_weights[k] =
    weights[cols[k]] * coeffs[k, :].sum()."""

    reduced: CpTensor
    cols: np.ndarray
    coeffs: np.ndarray
    new_weights: np.ndarray
    method: str
    numerical_rank: int
    rank_deficient: bool


def _assemble(x, decomp, method):
    """cp_tensor.py:215-232."""
    new_weights = x.weights[decomp.cols] * decomp.coeffs.sum(axis=1)
    reduced_weights = new_weights
    if decomp.rank_deficient:
        reduced_weights = new_weights.copy()
        reduced_weights[decomp.numerical_rank:] = 0.0
    reduced = x.select(decomp.cols, reduced_weights)
    return TensorIdResult(
        reduced=reduced, cols=decomp.cols, coeffs=decomp.coeffs, new_weights=new_weights,
        method=method, numerical_rank=decomp.numerical_rank,
        rank_deficient=decomp.rank_deficient,
    )


def tensor_id_from_sketch(x, sketch, rank, method, rank_tol=DEFAULT_RANK_TOL):
    """ID of a (host or device) sketch, then recombined weights (cp_tensor.py:235-239)."""
    decomp = matrix_id(sketch, rank, rank_tol=rank_tol)
    return _assemble(x, decomp, method)


def check_tensor_id_args(x, rank, sketch_dim, method):
    """cp_tensor.py:242-263."""
    if not 1 <= rank <= x.rank:
        raise ValueError(f"rank must be in [1, {x.rank}], got {rank}")
    if method == "gram":
        return None
    if sketch_dim is None:
        sketch_dim = rank + DEFAULT_OVERSAMPLE
    if sketch_dim < rank:
        raise ValueError(f"sketch dimension {sketch_dim} is below the target rank {rank}")
    if method == "tensorsketch" and sketch_dim >= x.total_entries:
        raise ValueError(f"sketch dimension {sketch_dim} must be < {x.total_entries} tensor entries")
    return sketch_dim


def tensorsketch_device(x, rank, sketch_dim=None, seed=None, rank_tol=DEFAULT_RANK_TOL):
    """Device half of tensorsketch_id: (DeviceId, sketch (R, L))."""
    sketch_dim = check_tensor_id_args(x, rank, sketch_dim, "tensorsketch")
    op = TensorSketchOp(x.mode_dims, sketch_dim, seed=seed)
    y, nrm = op.apply_device(x.factors, x.weights, norms=True)
    return device_matrix_id(y, sketch_dim, x.rank, rank, rank_tol, colnorm2=nrm), y


def tensorsketch_id(x, rank, sketch_dim=None, seed=None, rank_tol=DEFAULT_RANK_TOL):
    """Rank reduction via a TensorSketch of the flattened rank-1 terms
    (cp_tensor.py:266-276)."""
    res = _host_graph_call(x, rank, sketch_dim, seed, rank_tol)
    if res is not None:
        return res
    d, _ = tensorsketch_device(x, rank, sketch_dim, seed, rank_tol)
    return _assemble(x, d.to_host("tensorsketch"), "tensorsketch")


# Repeated tensorsketch_id calls on host tensors of one shape (trials,
# serving) replay a captured TensorIdGraph over persistent device copies of
# the factors: the second call with a given (mode dims, R, rank, L, rank_tol)
# captures it, later calls copy the factors and weights in (async DMA when
# the host memory is pinned), replay, and read (j, P) back in one copy.  The
# kernels and their order are the eager path's, so results are identical.
# One shape is kept; factors above HOST_GRAPH_MAX_BYTES always go eager.
HOST_GRAPHS = True
HOST_GRAPH_MAX_BYTES = 1 << 30
_host_graph = {"key": None, "seen": None, "graph": None, "bufs": None, "w": None, "stream": None}
_host_graph_lock = threading.Lock()


def _host_graph_call(x, rank, sketch_dim, seed, rank_tol):
    import torch

    from . import _device
    from .matrix_id import DeviceId

    if not HOST_GRAPHS or not all(isinstance(f, np.ndarray) for f in x.factors):
        return None
    if sum(f.nbytes for f in x.factors) > HOST_GRAPH_MAX_BYTES:
        return None
    L = check_tensor_id_args(x, rank, sketch_dim, "tensorsketch")
    from ._native import query

    if not query("ids_tensorsketch_fused_ok", len(x.mode_dims), L):
        return None  # the long-sketch (spectral) route is not captured
    key = (tuple(x.mode_dims), int(x.rank), int(rank), int(L), float(rank_tol),
           _device.device().index)
    # one caller at a time owns the cached graph and its buffers; concurrent
    # callers (other threads) take the eager path, which shares nothing
    if not _host_graph_lock.acquire(blocking=False):
        return None
    try:
        st = _host_graph
        if st["key"] != key:
            if st["seen"] != key:  # first sighting: the eager path this time
                st["seen"] = key
                return None
            st.update(key=None, graph=None, bufs=None, w=None, stream=None)
            try:
                bufs = [_device.empty((int(x.rank), d), torch.float64) for d in x.mode_dims]
                w = _device.empty(int(x.rank), torch.float64)
                _host_graph_fill(x, bufs, w)
                g = TensorIdGraph([b.t() for b in bufs], w, rank, L, rank_tol,
                                  host_weights=x.weights, split=True)
            except Exception:  # capture not possible here (e.g. memory): stay eager
                st["seen"] = ("no graph",) + key
                torch.cuda.synchronize()
                return None
            st.update(key=key, graph=g, bufs=bufs, w=w, stream=torch.cuda.Stream())
            g.host_out.copy_(g.device(seed), non_blocking=True)
        else:
            # the factor copies on a side stream, under the hash-draw replay
            g, side, main = st["graph"], st["stream"], torch.cuda.current_stream()
            side.wait_stream(main)  # buffers free, seeds and weights ordered
            with torch.cuda.stream(side):
                _host_graph_fill(x, st["bufs"], st["w"])
            g.host_out.copy_(g.device(seed, before_compute=lambda: main.wait_stream(side)),
                             non_blocking=True)
        torch.cuda.current_stream().synchronize()
        d = DeviceId.unpack(g.host_out.numpy(), int(rank), int(x.rank), "tensorsketch")
    finally:
        _host_graph_lock.release()
    return _assemble(x, d, "tensorsketch")


def _host_graph_fill(x, bufs, w):
    import torch

    for f, b in zip(x.factors, bufs):
        t = torch.from_numpy(f.T)  # F-order I_n x R -> contiguous (R, I_n)
        b.copy_(t, non_blocking=t.is_pinned())
    w.copy_(torch.from_numpy(np.ascontiguousarray(x.weights, dtype=np.float64)))


_TRIAL_SIDE = {}


def _trial_side_stream(device):
    import torch

    st = _TRIAL_SIDE.get(device)
    if st is None:
        st = _TRIAL_SIDE[device] = torch.cuda.Stream(device=device)
    return st


class TensorIdGraph:
    """tensorsketch_id of one device-resident CP tensor, captured once as a
    CUDA graph and replayed per seed (B200 extension; the reference has no
    counterpart -- its calls are host-bound numpy).

    Every kernel of the path -- the N per-mode hash draws (reading their
    PCG64 states from device memory, ids_countsketch_hash_dev), bucket
    indexes, scatter plans, the fused TensorSketch, the truncated CPQR and
    the coefficients -- is recorded once; a call writes the seed's per-mode
    states into a pinned buffer, copies them over (N x 32 bytes), replays the
    graph and reads (j, P) back in one packed copy.  Results are identical
    to tensorsketch_id on the same tensor and seed (same kernels, same
    order).

    factors: CUDA float64 I_n x R column-major (tensor.t() of an (R, I_n)
    contiguous tensor) -- normalized CP factors, as CpTensor stores them;
    weights: CUDA float64 (R,); host_weights: the same weights on the host
    (new_weights = weights[cols] * coeffs.sum(axis=1), cp_tensor.py:216, is
    formed in numpy, bit-identical to the reference).

    trials() of three or more seeds run on two split twins of the graph
    (pipeline_trials=True): the next trial's draw graph replays on a side
    stream beside the current trial's compute graph (C4 0.36 -> 0.32 ms per
    trial, C5 1.99 -> 1.93)."""

    def __init__(self, factors, weights, rank, sketch_dim=None, rank_tol=DEFAULT_RANK_TOL,
                 host_weights=None, split=False, pipeline_trials=True):
        import torch

        from . import _device

        import torch as _t

        if not all(isinstance(f, _t.Tensor) and f.device.type == "cuda" for f in factors) or \
                not (isinstance(weights, _t.Tensor) and weights.device.type == "cuda"):
            raise ValueError("TensorIdGraph takes CUDA factors and weights (host inputs cannot "
                             "be captured); use tensorsketch_id for host CP tensors")
        self.factors = [_fortran_cuda(f) for f in factors]
        self.weights = weights.to(_t.float64).contiguous()
        self.mode_dims = tuple(int(f.shape[0]) for f in self.factors)
        self.R = int(self.factors[0].shape[1])

        class _X:
            pass

        _X.rank = self.R
        _X.total_entries = int(np.prod(self.mode_dims))
        self.L = check_tensor_id_args(_X, rank, sketch_dim, "tensorsketch")
        self.k, self.rank_tol = int(rank), float(rank_tol)
        self.pipeline_trials, self._twin_graphs = bool(pipeline_trials), None
        self.host_weights = (np.asarray(host_weights, dtype=np.float64) if host_weights is not None
                             else weights.detach().cpu().numpy())
        n = len(self.mode_dims)
        self.seed_host = torch.empty((n, 4), dtype=torch.int64, pin_memory=True)
        self.seed_dev = _device.empty((n, 4), torch.int64)
        self.seed_host.numpy()[:] = TensorSketchOp.mode_seed_states(n, 0)
        self.seed_dev.copy_(self.seed_host)
        self._compute(self._draw())  # eager run: lazy initialization outside the capture
        torch.cuda.synchronize()
        lib = _device.lib()
        n0 = lib.ids_launch_count()
        # split=True: two graphs, the hash draws (which do not read the
        # factors) and the rest, so that a caller can refill the factors on
        # another stream while the draws replay (see _host_graph_call)
        self.graph = torch.cuda.CUDAGraph()
        self.graph_compute = torch.cuda.CUDAGraph() if split else None
        with torch.cuda.graph(self.graph, capture_error_mode="relaxed"):
            self._op = self._draw()
            if not split:
                self.out = self._compute(self._op)
        if split:
            with torch.cuda.graph(self.graph_compute, capture_error_mode="relaxed"):
                self.out = self._compute(self._op)
        self.launches = int(lib.ids_launch_count() - n0)  # library kernels per replay
        self.host_out = torch.empty(self.out.shape, dtype=self.out.dtype, pin_memory=True)

    PIPELINE_MIN_TRIALS = 3

    def _twins(self):
        if self._twin_graphs is None:
            mk = lambda: TensorIdGraph(self.factors, self.weights, self.k, self.L, self.rank_tol,
                                       host_weights=self.host_weights, split=True,
                                       pipeline_trials=False)
            self._twin_graphs = (mk(), mk())
        return self._twin_graphs

    def _draw(self):
        return TensorSketchOp(self.mode_dims, self.L, _seed_dev=self.seed_dev)

    def _compute(self, op):
        y, nrm = op.apply_device(self.factors, self.weights, norms=True)
        return device_matrix_id(y, self.L, self.R, self.k, self.rank_tol, colnorm2=nrm).packed()

    def device(self, seed, before_compute=None):
        """Replay for `seed`; the packed (cols, numerical rank, deficient, P)
        device vector (valid until the next replay).  before_compute (split
        graphs only): called between the two replays, e.g. to make the
        current stream wait for factor copies issued on another stream."""
        import torch

        self.seed_host.numpy()[:] = TensorSketchOp.mode_seed_states(len(self.mode_dims), seed)
        self.seed_dev.copy_(self.seed_host, non_blocking=True)
        self.graph.replay()
        if self.graph_compute is not None:
            if before_compute is not None:
                before_compute()
            self.graph_compute.replay()
        return self.out

    def trials(self, seeds):
        """[(InterpolativeDecomposition, new_weights)] for several seeds: one
        copy of every seed's states, the replays back to back (each result
        copied aside on the device), one device->host copy at the end."""
        import torch

        from . import _device
        from .matrix_id import DeviceId

        seeds = list(seeds)
        if not seeds:
            return []
        n = len(self.mode_dims)
        st = torch.from_numpy(np.stack([TensorSketchOp.mode_seed_states(n, s) for s in seeds]))
        st_dev = st.pin_memory().to(self.seed_dev.device, non_blocking=True)
        outs = []
        if len(seeds) >= TensorIdGraph.PIPELINE_MIN_TRIALS and self.pipeline_trials:
            # Two split twins of this graph (their own hash / plan / sketch
            # buffers) take the trials in turn: the next trial's draw graph
            # (hash draws, bucket indexes, scatter plans: short serial
            # kernels that leave the GPU idle) replays on a side stream
            # beside the current trial's compute graph.
            a, b = self._twins()
            main = torch.cuda.current_stream()
            side = _trial_side_stream(main.device)
            side.wait_stream(main)
            drawn = [None, None]
            computed = [None, None]

            def draw(t):
                g = (a, b)[t & 1]
                with torch.cuda.stream(side):
                    if computed[t & 1] is not None:  # the twin's last compute read its buffers
                        side.wait_event(computed[t & 1])
                    g.seed_dev.copy_(st_dev[t])
                    g.graph.replay()
                    ev = torch.cuda.Event()
                    ev.record()
                drawn[t & 1] = ev

            draw(0)
            for t in range(len(seeds)):
                if t + 1 < len(seeds):
                    draw(t + 1)
                g = (a, b)[t & 1]
                main.wait_event(drawn[t & 1])
                g.graph_compute.replay()
                outs.append(g.out.clone())
                ev = torch.cuda.Event()
                ev.record()
                computed[t & 1] = ev
            st_dev.record_stream(side)
        else:
            for t in range(len(seeds)):
                self.seed_dev.copy_(st_dev[t])
                self.graph.replay()
                if self.graph_compute is not None:
                    self.graph_compute.replay()
                outs.append(self.out.clone())
        host = _device.to_host(torch.stack(outs))
        res = []
        for v in host:
            d = DeviceId.unpack(v, self.k, self.R, "tensorsketch", copy=False)
            res.append((d, self.host_weights[d.cols] * d.coeffs.sum(axis=1)))
        return res

    def __call__(self, seed):
        """(InterpolativeDecomposition of the sketch, new_weights) for `seed`."""
        import torch

        from .matrix_id import DeviceId

        self.host_out.copy_(self.device(seed), non_blocking=True)
        torch.cuda.current_stream().synchronize()
        d = DeviceId.unpack(self.host_out.numpy(), self.k, self.R, "tensorsketch")
        return d, self.host_weights[d.cols] * d.coeffs.sum(axis=1)


# ---- error metric for tensor trials --------------------------
def _gram_device(weights, factor_lists):
    """diag(w) (hadamard of factor Grams) diag(w) on the device (cp_tensor.py:
    143-160).  Each entry of factor_lists is the list of column blocks of one
    mode (concatenated); the Grams are plain cuBLAS DGEMMs."""
    import torch

    from . import _device
    from .tensorsketch import factor_to_device

    out = None
    for blocks in factor_lists:
        t = torch.cat([factor_to_device(b) for b in blocks], 0)  # (R, I_n)
        g = t @ t.T
        out = g if out is None else out.mul_(g)
    w = _device.to_device(np.asarray(weights, dtype=np.float64), torch.float64)
    return out.mul_(w[None, :]).mul_(w[:, None])


def gram_hadamard(x):
    """Gram matrix of the flattened weighted rank-1 terms (cp_tensor.py:163-166)."""
    return _gram_device(x.weights, [[f] for f in x.factors]).cpu().numpy()


def cp_norm(x):
    """Exact Frobenius norm of a CP tensor via the Gram identity (cp_tensor.py:169-172)."""
    total = float(_gram_device(x.weights, [[f] for f in x.factors]).sum())
    return float(np.sqrt(max(total, 0.0)))


def cp_diff_norm(x, y):
    """Exact Frobenius norm of x - y for CP tensors (cp_tensor.py:183-197)."""
    if tuple(x.mode_dims) != tuple(y.mode_dims):
        raise ValueError(f"mode dimensions disagree: {x.mode_dims} vs {y.mode_dims}")
    weights = np.concatenate([x.weights, -np.asarray(y.weights)])
    total = float(_gram_device(weights, [[a, b] for a, b in zip(x.factors, y.factors)]).sum())
    return float(np.sqrt(max(total, 0.0)))


__all__ = [
    "CpTensor",
    "TensorIdGraph",
    "TENSOR_METHODS",
    "TensorIdResult",
    "check_tensor_id_args",
    "cp_diff_norm",
    "cp_norm",
    "gram_hadamard",
    "tensor_id_from_sketch",
    "tensorsketch_device",
    "tensorsketch_id",
]
