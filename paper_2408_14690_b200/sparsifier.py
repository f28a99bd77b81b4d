"""Magnitude sparsification and GPU histogram calibration.

Drop-in for pkg/src/actsparse/sparsifier.py:19-155 (same names, arguments,
error messages and numerics):

* the prune predicate is ``|x| <= t`` with a closed boundary, NaN kept,
  pruned entries written as +0.0; ``t`` is compared in fp32 after
  round-to-nearest, as NumPy's weak-scalar promotion does in the reference;
* histograms bin ``|x|`` in fp64 on the GPU with results bit-identical to the
  reference's numpy binning, and thresholds are inverted on the GPU with the
  reference's exact fp64 operation sequence.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _clib as C
from . import _runtime as RT

HISTOGRAM_MAGIC = "TEALH1"
DEFAULT_BIN_COUNT = 4096
HI_STD_MULTIPLE = 8.0


def _check_t(t) -> None:
    if not t >= 0.0:
        raise ValueError(f"threshold must be non-negative, got {t}")


def _device_input(x):
    """(flat CUDA tensor, original shape, host?) for numpy/list/torch input."""
    if isinstance(x, torch.Tensor) and x.is_cuda:
        xt = x if x.dtype in (torch.float32, torch.bfloat16) else x.float()
        return xt.contiguous().reshape(-1), tuple(x.shape), False
    dev = RT.require_cuda()
    a = np.asarray(x.cpu().numpy() if isinstance(x, torch.Tensor) else x, dtype=np.float32)
    return torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).to(dev), a.shape, True


def _hist_input(x):
    """Flat CUDA tensor for histogram binning: float64 stays float64 (host
    arrays are uploaded unrounded), fp32 / bf16 as they are."""
    if isinstance(x, torch.Tensor):
        if x.dtype == torch.float64:
            return x.to(RT.require_cuda() if not x.is_cuda else x.device).contiguous().reshape(-1)
        return _device_input(x)[0]
    a = np.asarray(x)
    if a.dtype == np.float64:
        return torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).to(RT.require_cuda())
    return _device_input(x)[0]


def threshold_bits(x, t: float):
    """(keep bitmask uint32 words, pruned count tensor) for a CUDA vector —
    bit i%32 of word i//32 is set iff !(|x_i| <= fl32(t))."""
    _check_t(t)
    xd, _, _ = _device_input(x)
    m = xd.numel()
    bits = torch.empty((m + 31) // 32, dtype=torch.int32, device=xd.device)
    pruned = torch.zeros(1, dtype=torch.int64, device=xd.device)
    C.call("teal_threshold", RT.ptr(xd), RT.dtype_code(xd.dtype), m, RT.f32_round_nearest(t),
           RT.ptr(bits), None, RT.ptr(pruned), RT.stream_handle())
    return bits, pruned


def sparsify(x, t: float):
    """Zero every entry with |x_i| <= t (closed boundary); keep the rest
    (sparsifier.py:120-125).  Host in -> host float32 out; CUDA in -> CUDA out."""
    _check_t(t)
    xd, shape, host = _device_input(x)
    out = torch.empty_like(xd)
    if xd.numel():
        C.call("teal_threshold", RT.ptr(xd), RT.dtype_code(xd.dtype), xd.numel(), RT.f32_round_nearest(t),
               None, RT.ptr(out), None, RT.stream_handle())
    out = out.reshape(shape)
    return out.cpu().numpy() if host else out


def realized_sparsity(x, t: float) -> float:
    """Fraction of entries with |x_i| <= t (sparsifier.py:128-133)."""
    xd, _, _ = _device_input(x)
    if xd.numel() == 0:
        raise ValueError("realized sparsity of an empty vector is undefined")
    t32 = RT.f32_round_nearest(t)
    if not t32 >= 0.0:  # no validation in the reference: |x| <= t holds nowhere
        return 0.0
    pruned = torch.zeros(1, dtype=torch.int64, device=xd.device)
    C.call("teal_threshold", RT.ptr(xd), RT.dtype_code(xd.dtype), xd.numel(), t32,
           None, None, RT.ptr(pruned), RT.stream_handle())
    return float(int(pruned.item())) / xd.numel()


def sparsify_batched(xs, t: float):
    """Shared-mask sparsification over a [B, m] batch (sparsifier.py:136-155):
    column i is zeroed in every row iff mean_b |X[b, i]| <= t."""
    _check_t(t)
    if isinstance(xs, torch.Tensor) and xs.is_cuda:
        batch, host = xs.float().contiguous(), False
        if batch.dim() != 2 or batch.shape[0] < 1:
            raise ValueError(f"expected a [B, m] batch with B >= 1, got shape {tuple(batch.shape)}")
    else:
        try:
            arr = np.asarray(xs, dtype=np.float32)
        except ValueError as exc:
            raise ValueError("ragged batch: all rows must have the same length") from exc
        if arr.ndim != 2 or arr.shape[0] < 1:
            raise ValueError(f"expected a [B, m] batch with B >= 1, got shape {arr.shape}")
        batch, host = torch.from_numpy(np.ascontiguousarray(arr)).to(RT.require_cuda()), True
    B, m = batch.shape
    out = torch.empty_like(batch)
    mask = torch.empty(m, dtype=torch.uint8, device=batch.device)
    C.call("teal_threshold_batched", RT.ptr(batch), B, m, RT.f32_round_nearest(t), RT.ptr(mask), RT.ptr(out),
           RT.stream_handle())
    if host:
        return out.cpu().numpy(), mask.cpu().numpy().astype(bool)
    return out, mask.bool()


class DistFamily(Enum):
    GAUSSIAN = "gaussian"
    LAPLACE = "laplace"


class ActivationHistogram:
    """Per-layer histogram of activation magnitudes with device-resident
    int64 counts (sparsifier.py:30-117).

    Uniform bins on [0, hi], last bin closed at hi, |x| > hi -> overflow.
    ``record`` bins on the GPU in fp64; ``threshold`` inverts on the GPU."""

    def __init__(self, layer_id: str, bin_count: int, lo: float, hi: float, counts,
                 overflow_count: int = 0, total: int = 0):
        if bin_count < 1:
            raise ValueError(f"bin_count must be >= 1, got {bin_count}")
        if lo != 0.0:
            raise ValueError("histogram lower bound must be 0 (magnitudes)")
        if not hi > 0:
            raise ValueError(f"histogram upper bound must be positive, got {hi}")
        c = counts.detach().cpu().numpy() if isinstance(counts, torch.Tensor) else np.asarray(counts)
        c = c.astype(np.int64)
        if c.shape != (bin_count,):
            raise ValueError("counts length must equal bin_count")
        if (c < 0).any() or overflow_count < 0:
            raise ValueError("negative bin counts")
        if total != int(c.sum()) + overflow_count:
            raise ValueError("total != sum(counts) + overflow_count")
        self.layer_id = layer_id
        self.bin_count = int(bin_count)
        self.lo = 0.0
        self.hi = float(hi)
        self.overflow_count = int(overflow_count)
        self.total = int(total)
        self._counts_host = c
        self._dev = None  # (counts int64 [bins], overflow int64 [1]) on device, authoritative when set

    @classmethod
    def empty(cls, layer_id: str, bin_count: int, hi: float) -> "ActivationHistogram":
        return cls(layer_id, bin_count, 0.0, float(hi), np.zeros(bin_count, dtype=np.int64), 0, 0)

    # -- device state ------------------------------------------------------------
    def _device_state(self, device):
        if self._dev is None or self._dev[0].device != device:
            counts = torch.from_numpy(self._counts_host.copy()).to(device)
            ov = torch.tensor([self.overflow_count], dtype=torch.int64, device=device)
            self._dev = (counts, ov)
        return self._dev

    @property
    def counts(self) -> np.ndarray:
        if self._dev is not None:
            self._counts_host = self._dev[0].cpu().numpy()
        return self._counts_host.copy()

    def record(self, x) -> "ActivationHistogram":
        """Add |x_i| for every entry of x; values above hi count as overflow.
        NaN input raises ValueError and leaves the histogram unchanged.
        float64 input is binned at float64 (the reference's np.asarray(x,
        float64), sparsifier.py:75-80), everything else at its own precision."""
        xd = _hist_input(x)
        n = xd.numel()
        if n == 0:
            return self
        counts, ov = self._device_state(xd.device)
        dcounts = torch.zeros_like(counts)
        dov = torch.zeros(1, dtype=torch.int64, device=xd.device)
        flag = torch.zeros(1, dtype=torch.int32, device=xd.device)
        C.call("teal_hist_record", RT.ptr(xd), RT.dtype_code(xd.dtype), n, self.hi, self.bin_count,
               RT.ptr(dcounts), RT.ptr(dov), RT.ptr(flag), RT.stream_handle())
        if int(flag.item()):
            raise ValueError("cannot record NaN activations")
        counts += dcounts
        ov += dov
        self.overflow_count = int(ov.item())
        self.total += n
        return self

    def merge(self, other: "ActivationHistogram") -> "ActivationHistogram":
        if (other.bin_count, other.lo, other.hi) != (self.bin_count, self.lo, self.hi):
            raise ValueError("cannot merge histograms with different binning")
        dev = self._dev[0].device if self._dev is not None else RT.require_cuda()
        counts, ov = self._device_state(dev)
        oc, oo = other._device_state(dev)
        counts += oc
        ov += oo
        self.overflow_count += other.overflow_count
        self.total += other.total
        return self

    def thresholds(self, ps) -> list[float]:
        """Batch form of :meth:`threshold` (one GPU launch)."""
        ps = [float(p) for p in ps]
        for p in ps:
            if not 0.0 <= p <= 1.0:
                raise ValueError(f"sparsity must lie in [0, 1], got {p}")
        if self.total < 1:
            raise ValueError("cannot estimate a threshold from an empty histogram")
        if not ps:
            return []
        dev = self._dev[0].device if self._dev is not None else RT.require_cuda()
        counts, ov = self._device_state(dev)
        pd = torch.tensor(ps, dtype=torch.float64, device=dev)
        out = torch.empty(len(ps), dtype=torch.float64, device=dev)
        C.call("teal_hist_threshold", RT.ptr(counts), self.bin_count, RT.ptr(ov), self.hi, RT.ptr(pd), len(ps),
               RT.ptr(out), RT.stream_handle())
        return [float(v) for v in out.cpu().tolist()]

    def threshold(self, p: float) -> float:
        """Smallest bin-interpolated t with empirical CDF(t) >= p
        (sparsifier.py:94-117); p=0 -> 0, p=1 -> hi."""
        return self.thresholds([p])[0]

    def __repr__(self):
        return (f"ActivationHistogram(layer_id={self.layer_id!r}, bin_count={self.bin_count}, "
                f"hi={self.hi!r}, total={self.total}, overflow_count={self.overflow_count})")


# --- histogram file format (sparsifier.py:189-219), byte-compatible ------------

def save_histogram(path: str | os.PathLike, hist: ActivationHistogram) -> None:
    if any(ch.isspace() for ch in hist.layer_id):
        raise ValueError(f"layer_id must not contain whitespace: {hist.layer_id!r}")
    lines = [f"{HISTOGRAM_MAGIC} {hist.layer_id} {hist.bin_count} "
             f"{hist.lo:.17g} {hist.hi:.17g} {hist.total} {hist.overflow_count}"]
    lines.extend(str(int(c)) for c in hist.counts)
    with open(path, "w", encoding="ascii") as fh:
        fh.write("\n".join(lines))
        fh.write("\n")


def load_histogram(path: str | os.PathLike) -> ActivationHistogram:
    with open(path, "r", encoding="ascii") as fh:
        header = fh.readline().strip().split()
        if len(header) != 7 or header[0] != HISTOGRAM_MAGIC:
            raise ValueError(f"bad histogram header in {path}")
        layer_id, bin_count = header[1], int(header[2])
        lo, hi = float(header[3]), float(header[4])
        total, overflow = int(header[5]), int(header[6])
        counts = np.array([int(fh.readline()) for _ in range(bin_count)], dtype=np.int64)
    return ActivationHistogram(layer_id, bin_count, lo, hi, counts, overflow, total)


@dataclass(frozen=True)
class DistributionFit:
    family: DistFamily
    location: float
    scale: float
    neg_log_likelihood: float
