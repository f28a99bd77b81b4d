"""Layout-tagged matrices with device-resident input-major storage, seeded
sampling, and the dense GEMV.

Drop-in for the reference substrate (pkg/src/actsparse/tensor.py:30-194):
same names, constructor arguments, validation messages and layout contract
(element (i, j) at ``i*cols + j`` under ROW_MAJOR and ``j*rows + i`` under
COL_MAJOR, tensor.py:47-48).  The difference is where the bytes live: a
:class:`Matrix` uploads its data once to HBM in input-channel-major order
(``[cols][rows]`` = the COL_MAJOR flat buffer) and keeps it resident; every
product runs in the sm_100a library.
"""

from __future__ import annotations

from enum import Enum

import numpy as np
import torch

from . import _clib as C
from . import _runtime as RT

WEIGHT_MAGIC = "TEALW1"
_CHILD_TAG = 0x9E3779B9


class Layout(Enum):
    ROW_MAJOR = "rowmajor"
    COL_MAJOR = "colmajor"


def as_vector(x) -> np.ndarray:
    """1-D float32 host vector (tensor.py:33-38)."""
    v = np.asarray(x, dtype=np.float32)
    if v.ndim != 1:
        raise ValueError(f"expected a 1-D vector, got shape {v.shape}")
    return v


class Matrix:
    """2-D matrix with an explicit physical layout (tensor.py:41-96).

    Host construction mirrors the reference (flat float32 ``data``, made
    read-only).  :meth:`from_device` wraps weights that already live in HBM
    in input-major order (``[m_in, n_out]`` = COL_MAJOR), in float32, bfloat16
    or int8 (with a per-output-column fp32 scale)."""

    __slots__ = ("rows", "cols", "layout", "_data", "_dev", "_scale")

    def __init__(self, rows: int, cols: int, layout: Layout, data):
        if rows < 1 or cols < 1:
            raise ValueError(f"invalid matrix shape {rows}x{cols}")
        if not isinstance(data, np.ndarray) or data.dtype != np.float32 or data.ndim != 1:
            raise ValueError("matrix data must be a flat float32 array")
        if data.size != rows * cols:
            raise ValueError(f"data length {data.size} does not match rows*cols = {rows * cols}")
        data.flags.writeable = False
        self.rows, self.cols, self.layout = int(rows), int(cols), layout
        self._data = data
        self._dev = {}
        self._scale = None

    # -- construction -------------------------------------------------------
    @classmethod
    def from_2d(cls, arr, layout: Layout = Layout.ROW_MAJOR) -> "Matrix":
        a = np.asarray(arr, dtype=np.float32)
        if a.ndim != 2:
            raise ValueError(f"expected a 2-D array, got shape {a.shape}")
        flat = np.array(a.ravel(order="C" if layout is Layout.ROW_MAJOR else "F"), copy=True)
        return cls(a.shape[0], a.shape[1], layout, flat)

    @classmethod
    def from_device(cls, w_in_major: torch.Tensor, col_scale: torch.Tensor | None = None) -> "Matrix":
        """Wrap a resident ``[m_in, n_out]`` CUDA tensor (logical W is [n_out, m_in])."""
        if w_in_major.dim() != 2 or not w_in_major.is_cuda:
            raise ValueError("from_device expects a 2-D CUDA tensor [m_in, n_out]")
        if w_in_major.dtype not in (torch.float32, torch.bfloat16, torch.int8):
            raise ValueError(f"unsupported weight dtype {w_in_major.dtype}")
        if (w_in_major.dtype == torch.int8) != (col_scale is not None):
            raise ValueError("int8 weights need (and only int8 weights take) a per-column scale")
        m, n = w_in_major.shape
        obj = cls.__new__(cls)
        obj.rows, obj.cols, obj.layout = int(n), int(m), Layout.COL_MAJOR
        obj._data = None
        obj._dev = {(w_in_major.device, w_in_major.dtype): w_in_major.contiguous()}
        obj._scale = col_scale.contiguous().to(torch.float32) if col_scale is not None else None
        return obj

    # -- views ----------------------------------------------------------------
    @property
    def data(self) -> np.ndarray:
        if self._data is None:
            d = self.to_2d().ravel(order="F")
            d.flags.writeable = False
            self._data = d
        return self._data

    def to_2d(self) -> np.ndarray:
        """Logical [rows, cols] host array."""
        if self._data is not None:
            order = "C" if self.layout is Layout.ROW_MAJOR else "F"
            return self._data.reshape((self.rows, self.cols), order=order)
        (dev_dt, t), = list(self._dev.items())[:1]
        w = t.float()
        if self._scale is not None:
            w = w * self._scale[None, :]
        return w.t().contiguous().cpu().numpy()

    def at(self, i: int, j: int) -> float:
        return float(self.to_2d()[i, j])

    @property
    def device_dtype(self) -> torch.dtype:
        if self._data is None:
            return next(iter(self._dev))[1]
        return torch.float32

    @property
    def col_scale(self):
        return self._scale

    def in_major(self, device=None, dtype: torch.dtype | None = None) -> torch.Tensor:
        """Resident input-major ``[cols, rows]`` copy on ``device`` (cached)."""
        device = torch.device(device) if device is not None else RT.require_cuda()
        if device.index is None:
            device = torch.device("cuda", torch.cuda.current_device())
        dtype = dtype or self.device_dtype
        key = (device, dtype)
        t = self._dev.get(key)
        if t is None:
            if self._data is None:
                src = next(iter(self._dev.values()))
                if src.dtype == torch.int8:
                    raise ValueError("int8 matrices cannot be re-typed")
                t = src.to(device=device, dtype=dtype).contiguous()
            else:
                host = self.to_2d().T  # [cols, rows] logical transpose = input-major
                t = torch.from_numpy(np.ascontiguousarray(host)).to(device=device, dtype=dtype)
            self._dev[key] = t
        return t


def to_layout(w: Matrix, layout: Layout) -> Matrix:
    """Bit-exact re-store under a new layout (tensor.py:86-91)."""
    if w.layout is layout:
        return w
    order = "C" if layout is Layout.ROW_MAJOR else "F"
    return Matrix(w.rows, w.cols, layout, np.array(w.to_2d().ravel(order=order), copy=True))


# ---- dense GEMV -----------------------------------------------------------------

def _to_device_vector(x, device):
    """(device fp32/bf16 vector, was_host) for a host array or CUDA tensor."""
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            return x.to(device=device, dtype=torch.float32).reshape(-1).contiguous(), True
        if x.dim() != 1:
            raise ValueError(f"expected a 1-D vector, got shape {tuple(x.shape)}")
        if x.dtype not in (torch.float32, torch.bfloat16):
            x = x.float()
        return x.contiguous(), False
    v = as_vector(x)
    return torch.from_numpy(np.ascontiguousarray(v)).to(device, non_blocking=False), True


def _gemv(w: Matrix, xd: torch.Tensor, t32: float, kept=None, out=None) -> torch.Tensor:
    dev = xd.device
    wt = w.in_major(dev)
    m, n = w.cols, w.rows
    y = out if out is not None else torch.empty(n, dtype=torch.float32, device=dev)
    a = RT.single_gemv_args(wt, n, xd, float(t32), y, w.col_scale, kept)
    RT.bind_workspace(a, dev)
    RT.launch_gemv(a)
    return y


def matmul_dense(x, w: Matrix):
    """y = x W^T for x of length w.cols (tensor.py:130-140), on the GPU.

    Host input -> host float32 result; CUDA input -> CUDA result."""
    dev = RT.require_cuda() if not (isinstance(x, torch.Tensor) and x.is_cuda) else x.device
    size = x.numel() if isinstance(x, torch.Tensor) else np.asarray(x).size
    if isinstance(x, torch.Tensor) and x.dim() != 1:
        raise ValueError(f"expected a 1-D vector, got shape {tuple(x.shape)}")
    if size != w.cols:
        raise ValueError(
            f"dimension mismatch: x has length {size}, W is {w.rows}x{w.cols} "
            f"(expected x length {w.cols})")
    xd, host = _to_device_vector(x, dev)
    y = _gemv(w, xd, float("-inf"))
    return y.cpu().numpy() if host else y


# ---- seeded sampling (tensor.py:143-194) ------------------------------------------

class RngStream:
    """Counter-based deterministic stream: each draw is a Philox generator keyed
    by SeedSequence(seed, spawn_key=(counter,)) (tensor.py:146-171), so the
    same seeds give the reference's exact inputs and weights."""

    __slots__ = ("seed", "counter")

    def __init__(self, seed: int, counter: int = 0):
        self.seed = int(seed)
        self.counter = int(counter)

    def _entropy(self) -> int:
        return self.seed & 0xFFFF_FFFF_FFFF_FFFF

    def next_generator(self) -> np.random.Generator:
        ss = np.random.SeedSequence(entropy=self._entropy(), spawn_key=(self.counter,))
        self.counter += 1
        return np.random.Generator(np.random.Philox(ss))

    def child(self, index: int) -> "RngStream":
        ss = np.random.SeedSequence(entropy=self._entropy(), spawn_key=(_CHILD_TAG, int(index)))
        return RngStream(int(ss.generate_state(1, np.uint64)[0]))

    def __repr__(self):
        return f"RngStream(seed={self.seed}, counter={self.counter})"


def sample_gaussian(rng: RngStream, n: int, sigma: float) -> np.ndarray:
    if n < 1:
        raise ValueError(f"need n >= 1, got {n}")
    if not sigma > 0:
        raise ValueError(f"sigma must be positive, got {sigma}")
    return rng.next_generator().standard_normal(n, dtype=np.float32) * np.float32(sigma)


def sample_laplace(rng: RngStream, n: int, scale: float) -> np.ndarray:
    if n < 1:
        raise ValueError(f"need n >= 1, got {n}")
    if not scale > 0:
        raise ValueError(f"scale must be positive, got {scale}")
    return (rng.next_generator().laplace(0.0, 1.0, size=n) * scale).astype(np.float32)


# ---- weight file TEALW1 (tensor.py:197-235), byte-compatible ----------------------
#
# Header b"TEALW1 <rows> <cols> <layout>\n" then rows*cols little-endian f32 in
# logical row-major order whatever the layout; the round trip is bit-exact, so
# weights written by the reference CLI load straight into HBM here.

def write_matrix(fh, w: Matrix) -> None:
    fh.write(f"{WEIGHT_MAGIC} {w.rows} {w.cols} {w.layout.value}\n".encode("ascii"))
    fh.write(np.ascontiguousarray(w.to_2d(), dtype="<f4").tobytes(order="C"))


def read_matrix(fh) -> Matrix:
    header = fh.readline().decode("ascii", errors="replace").strip()
    parts = header.split()
    if len(parts) != 4 or parts[0] != WEIGHT_MAGIC:
        raise ValueError(f"bad weight header: {header!r}")
    rows, cols = int(parts[1]), int(parts[2])
    try:
        layout = Layout(parts[3])
    except ValueError:
        raise ValueError(f"unknown layout tag {parts[3]!r} in weight header") from None
    nbytes = rows * cols * 4
    payload = fh.read(nbytes)
    if len(payload) != nbytes:
        raise ValueError(f"truncated weight payload: expected {nbytes} bytes, got {len(payload)}")
    arr = np.frombuffer(payload, dtype="<f4").astype(np.float32).reshape(rows, cols)
    return Matrix.from_2d(arr, layout)


def save_matrix(path, w: Matrix) -> None:
    with open(path, "wb") as fh:
        write_matrix(fh, w)


def load_matrix(path) -> Matrix:
    with open(path, "rb") as fh:
        return read_matrix(fh)
