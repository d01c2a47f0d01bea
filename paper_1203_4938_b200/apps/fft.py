"""FFT application API on the B200 nodes (mirror of dpp.apps.fft).

Same names and argument meaning as /root/reference/pkg/src/dpp/apps/fft.py:
``FftPlan`` (fft.py:126-147), ``fft`` (fft.py:150-174), ``leaf_kernel`` /
``leaf_program`` (fft.py:86-123), ``bit_reverse_indices`` (fft.py:45-53),
``fft_bench`` / ``BenchRow`` / ``parse_sizes`` (fft.py:180-262).

What changes is where the work runs.  The reference permutes on the host,
ships 2^k-point leaves to the engine and finishes log2(N)-k butterfly stages
on the host in binary64.  Here the whole transform is ONE graph node,
``fft{N}`` (``fft_program``), executed by the sm_100a Stockham/four-step
kernels; ``leaf_program`` nodes still run natively (bit-exact with the
reference engine) for graphs that use them.  ``fft2`` adds the 2-D transform
(rows then columns) the reference lacks.

The ``fft{N}`` node's body is a valid kernel-language naive DFT, so the same
document also runs on the reference engine (slowly) and names its meaning.
"""

from __future__ import annotations

import functools
import os
import threading

from dataclasses import dataclass, replace

import numpy as np

from ..client import CudaBackend, run
from ..model import Instance, Node, Program, frozen_program
from ..types import DataType, Direction, IOPoint
from ..wire import DeviceStream, StreamFile

__all__ = ["MAX_LEAF_ORDER", "FftPlan", "fft", "fft_batch", "fft2", "naive_dft", "bit_reverse_indices",
           "leaf_kernel", "leaf_program", "fft_kernel", "fft_program", "fft2d_kernel",
           "fft2d_program", "fft_bench", "BenchRow", "parse_sizes", "NATIVE_TAG"]

MAX_LEAF_ORDER = 3
NATIVE_TAG = "// dpp-b200 native:"


def naive_dft(signal) -> np.ndarray:
    """Direct O(N^2) DFT (fft.py:32-42) computed on the device in binary64 and
    rounded to complex64; numpy in -> numpy out, CUDA tensor in -> tensor out."""
    import torch

    from .. import _lib
    from .._torch import require_cuda, stream_handle
    is_t = isinstance(signal, torch.Tensor)
    x = signal if is_t else torch.from_numpy(np.ascontiguousarray(signal, np.complex64))
    if x.numel() < 1:
        raise ValueError("signal must have at least one sample")
    dev = x.device if is_t and x.is_cuda else require_cuda(None)
    xd = x.to(dev, torch.complex64).contiguous()
    n = xd.shape[-1]
    y = torch.empty_like(xd)
    _lib.check(_lib.load().dpp_naive_dft(xd.data_ptr(), y.data_ptr(), n, xd.numel() // n, stream_handle()),
               "naive_dft")
    return y if is_t and x.is_cuda else y.cpu().numpy()


def bit_reverse_indices(n: int) -> np.ndarray:
    """Index i -> bit-reversed i over log2(n) bits (fft.py:45-53)."""
    bits = int(n).bit_length() - 1
    idx = np.arange(n, dtype=np.int64)
    rev = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        rev |= ((idx >> b) & 1) << (bits - 1 - b)
    return rev


# ---------------------------------------------------------------------------
# node bodies

def _unit_coeff(t: int, size: int) -> tuple[float, float]:
    a = -2.0 * np.pi * (t % size) / size
    c, s = float(np.cos(a)), float(np.sin(a))
    snap = lambda v: next((e for e in (-1.0, 0.0, 1.0) if abs(v - e) < 1e-12), v)  # noqa: E731
    return snap(c), snap(s)


def _literal_term(coeff: float, operand: str) -> str:
    if coeff == 0.0:
        return ""
    sign = "-" if coeff < 0 else "+"
    if abs(coeff) == 1.0:
        return f"{sign} {operand}"
    text = np.format_float_positional(np.float32(abs(coeff)), unique=True)
    return f"{sign} {text}f*{operand}"


def _join(terms: list[str]) -> str:
    s = " ".join(t for t in terms if t)
    return s[2:] if s.startswith("+ ") else s


def leaf_kernel(k: int) -> Node:
    """dft{2^k}: one dense 2^k-point DFT per float{2^(k+1)} work-item (fft.py:86-117).

    The generated text is identical to the reference's, so the native
    registry recognises reference-built leaf programs byte for byte."""
    if not 1 <= k <= MAX_LEAF_ORDER:
        raise ValueError(f"leaf order must be 1..{MAX_LEAF_ORDER}, got {k}")
    size, width = 1 << k, 2 << k
    pos = bit_reverse_indices(size)
    exprs = []
    for j in range(size):
        re, im = [], []
        for n in range(size):
            c, s = _unit_coeff(j * n, size)
            at = int(pos[n])
            xr, xi = f"v.s{2 * at:x}", f"v.s{2 * at + 1:x}"
            re += [_literal_term(c, xr), _literal_term(-s, xi)]
            im += [_literal_term(s, xr), _literal_term(c, xi)]
        exprs += [_join(re), _join(im)]
    body = (f"int i = get_global_id(0);\nfloat{width} v = x[i];\n"
            f"y[i] = (float{width})(\n    " + ",\n    ".join(exprs) + ");\n")
    dt = DataType("float", width)
    return Node(f"dft{size}", body, (IOPoint("x", dt, Direction.INPUT),
                                      IOPoint("y", dt, Direction.OUTPUT)))


def leaf_program(k: int) -> Program:
    node = leaf_kernel(k)
    return Program({node.name: node}, (Instance(0, node.name),), ())


def fft_kernel(n: int) -> Node:
    """Whole-transform node ``fft{n}``: x, y float2 (one complex sample per
    work-item); every run of n consecutive work-items is one signal, so the
    chunk must hold whole signals.  Body = naive DFT in the kernel language
    (valid on the reference engine; executed natively here)."""
    FftPlan(n, 1)
    body = (f"{NATIVE_TAG} fft n={n}\n"
            "int i = get_global_id(0);\n"
            f"int k = i % {n};\n"
            "int base = i - k;\n"
            "float re = 0.0f;\n"
            "float im = 0.0f;\n"
            f"for (int j = 0; j < {n}; j = j + 1) {{\n"
            f"    long ph = ((long)(k) * (long)(j)) % {n};\n"
            f"    float a = -2.0f * M_PI_F * (float)(ph) / {n}.0f;\n"
            "    float2 v = x[base + j];\n"
            "    float c = cos(a);\n"
            "    float s = sin(a);\n"
            "    re = re + v.x * c - v.y * s;\n"
            "    im = im + v.x * s + v.y * c;\n"
            "}\n"
            "y[i] = (float2)(re, im);\n")
    dt = DataType("float", 2)
    return Node(f"fft{n}", body, (IOPoint("x", dt, Direction.INPUT), IOPoint("y", dt, Direction.OUTPUT)))


@functools.lru_cache(maxsize=64)
def _fft_program_cached(n: int) -> Program:
    node = fft_kernel(n)
    return frozen_program(Program({node.name: node}, (Instance(0, node.name),), ()))


def fft_program(n: int) -> Program:
    """One-instance program with the fft{n} node (built once per n and shared;
    its id is computed once)."""
    return _fft_program_cached(n)


def fft2d_kernel(rows: int, cols: int) -> Node:
    """2-D node ``fft2d_{rows}x{cols}``: x, y float2 in row-major images of
    rows*cols work-items (naive 2-D DFT body; native: row + column passes)."""
    FftPlan(rows, 1)
    FftPlan(cols, 1)
    size = rows * cols
    body = (f"{NATIVE_TAG} fft2d rows={rows} cols={cols}\n"
            "int i = get_global_id(0);\n"
            f"int off = i % {size};\n"
            "int base = i - off;\n"
            f"int ku = off / {cols};\n"
            f"int kv = off % {cols};\n"
            "float re = 0.0f;\n"
            "float im = 0.0f;\n"
            f"for (int u = 0; u < {rows}; u = u + 1) {{\n"
            f"    for (int v = 0; v < {cols}; v = v + 1) {{\n"
            f"        long pu = ((long)(ku) * (long)(u)) % {rows};\n"
            f"        long pv = ((long)(kv) * (long)(v)) % {cols};\n"
            f"        float a = -2.0f * M_PI_F * ((float)(pu) / {rows}.0f + (float)(pv) / {cols}.0f);\n"
            f"        float2 s = x[base + u * {cols} + v];\n"
            "        re = re + s.x * cos(a) - s.y * sin(a);\n"
            "        im = im + s.x * sin(a) + s.y * cos(a);\n"
            "    }\n"
            "}\n"
            "y[i] = (float2)(re, im);\n")
    dt = DataType("float", 2)
    return Node(f"fft2d_{rows}x{cols}", body,
                (IOPoint("x", dt, Direction.INPUT), IOPoint("y", dt, Direction.OUTPUT)))


def fft2d_program(rows: int, cols: int) -> Program:
    node = fft2d_kernel(rows, cols)
    return Program({node.name: node}, (Instance(0, node.name),), ())


# ---------------------------------------------------------------------------
# plan + transforms

@dataclass(frozen=True)
class FftPlan:
    """Transform size plus leaf order (fft.py:126-147); ``k`` only matters for
    leaf programs, the native transform is radix-16 regardless."""

    n: int
    k: int = MAX_LEAF_ORDER

    def __post_init__(self) -> None:
        if self.n < 2 or self.n & (self.n - 1):
            raise ValueError(f"transform size must be a power of two, got {self.n}")
        if not 1 <= self.k <= MAX_LEAF_ORDER:
            raise ValueError(f"leaf order must be 1..{MAX_LEAF_ORDER}")
        if 2 ** self.k > self.n:
            raise ValueError(f"leaf size {2 ** self.k} exceeds transform size {self.n}")

    @property
    def leaf_size(self) -> int:
        return 2 ** self.k

    @property
    def vector_width(self) -> int:
        return 2 * self.leaf_size


def _as_stream(x, count_check: int):
    """Host complex64 array or CUDA complex64 tensor -> (input stream, is_device)."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if x.dtype != torch.complex64:
                raise ValueError(f"expected complex64, got {x.dtype}")
            flat = torch.view_as_real(x.contiguous()).reshape(-1)
            return DeviceStream(DataType("float", 2), flat), True
    except ImportError:  # pragma: no cover
        pass
    arr = np.ascontiguousarray(x, np.complex64)
    return StreamFile(DataType("float", 2), arr.reshape(-1).view(np.float32)), False


def _backend_for(backend, device_input: bool) -> CudaBackend:
    backend = backend or CudaBackend()
    return replace(backend, outputs="device") if device_input else backend


def _unstream(sf, shape, device: bool):
    if device:
        import torch
        return torch.view_as_complex(sf.tensor.view(-1, 2)).reshape(shape)
    return sf.values.view(np.complex64).reshape(shape)


def fft(signal, fft_plan: FftPlan | None = None, backend: CudaBackend | None = None):
    """Forward FFT of one complex64 signal (fft.py:150-174) through ``fft{N}``.

    Accepts a numpy array (returns numpy) or a CUDA complex64 tensor
    (returns a CUDA tensor; nothing crosses the bus)."""
    n = len(signal)
    fft_plan = fft_plan or FftPlan(n)
    if fft_plan.n != n:
        raise ValueError(f"plan is for {fft_plan.n} samples, got {n}")
    return fft_batch(signal, fft_plan.n, backend, _shape=(n,))


def fft_batch(signals, n: int | None = None, backend: CudaBackend | None = None, *, out=None,
              _shape=None):
    """Forward FFT of every row of a (batch, n) complex64 array/tensor.

    numpy in -> numpy out; CUDA tensor in -> CUDA tensor out (no transfer);
    CPU (ideally pinned) tensor in -> CPU tensor out, written into ``out``
    when given: H2D, transform and D2H are stream-ordered, one sync at the end."""
    shape = tuple(signals.shape) if _shape is None else _shape
    n = shape[-1] if n is None else n
    FftPlan(n, 1)
    if shape[-1] != n:
        raise ValueError(f"plan is for {n} samples, got {shape[-1]}")
    import torch
    if isinstance(signals, torch.Tensor) and not signals.is_cuda:
        from .._torch import require_cuda
        dev = require_cuda((backend or CudaBackend()).device)
        out = torch.empty(shape, dtype=torch.complex64, pin_memory=True) if out is None else out
        if signals.is_pinned() and out.is_pinned() and signals.is_contiguous() and out.is_contiguous():
            return _fft_host_pipelined(signals, n, out, dev)
        d_in = signals.to(dev, non_blocking=signals.is_pinned())
        d_out = fft_batch(d_in, n, backend, _shape=shape)
        out.copy_(d_out, non_blocking=out.is_pinned())
        torch.cuda.current_stream(dev).synchronize()
        return out
    stream, dev = _as_stream(signals, n)
    backend = _backend_for(backend, dev)
    if not dev and backend.chunk_size is None and stream.values.nbytes > _PIPE_CHUNK_BYTES:
        # large host batches: whole signals per chunk, so the engine pipelines
        # H2D / transform / D2H over max_in_flight device slots (client.run)
        backend = replace(backend, chunk_size=max(1, _PIPE_CHUNK_BYTES // (8 * n)) * n)
    out = run(backend, fft_program(n), {"0.x": stream})["0.y"]
    return _unstream(out, shape, isinstance(out, DeviceStream))


_PIPE_CHUNK_BYTES = int(os.environ.get("DPP_PIPE_CHUNK_MB", "128")) << 20
_pipes: dict = {}
_pipes_lock = threading.Lock()


def _fft_host_pipelined(signals, n: int, out, dev):
    """Pinned host -> device -> FFT -> pinned host, in chunks on three streams.

    H2D of chunk c+1, the transform of chunk c and the D2H of chunk c-1 run
    concurrently (PCIe is full duplex), so the host round trip the paper names
    as the GPU bottleneck costs max(H2D, D2H) instead of
    their sum.  Three rotating device slots; transforms run in place.  A
    pipeline (streams + slots) is shared per (device, chunk, n) and owned by
    one caller at a time."""
    import torch

    rows = signals.numel() // n
    src = signals.reshape(rows, n)
    dst = out.reshape(rows, n)
    per = max(1, min(rows, _PIPE_CHUNK_BYTES // (8 * n)))
    key = (dev.index, per, n)
    with _pipes_lock:
        st = _pipes.get(key)
        if st is None:
            st = {"h2d": torch.cuda.Stream(dev), "fft": torch.cuda.Stream(dev), "d2h": torch.cuda.Stream(dev),
                  "bufs": [torch.empty((per, n), dtype=torch.complex64, device=dev) for _ in range(3)],
                  "loaded": [torch.cuda.Event() for _ in range(3)], "done": [torch.cuda.Event() for _ in range(3)],
                  "free": [None, None, None], "lock": threading.Lock()}
            _pipes[key] = st
    with st["lock"]:  # one caller at a time owns the pipeline's streams and slots
        return _run_pipe(st, src, dst, rows, per, n, dev, out)


def _run_pipe(st, src, dst, rows, per, n, dev, out):
    import torch

    from .. import ops
    caller = torch.cuda.current_stream(dev)
    st["h2d"].wait_stream(caller)
    for c, r0 in enumerate(range(0, rows, per)):
        k = c % 3
        m = min(per, rows - r0)
        buf = st["bufs"][k][:m]
        if st["free"][k] is not None:
            st["h2d"].wait_event(st["free"][k])
        with torch.cuda.stream(st["h2d"]):
            buf.copy_(src[r0:r0 + m], non_blocking=True)
            st["loaded"][k].record(st["h2d"])
        st["fft"].wait_event(st["loaded"][k])
        ops.fft_forward(buf, n, out=buf, stream=st["fft"])
        st["done"][k].record(st["fft"])
        st["d2h"].wait_event(st["done"][k])
        with torch.cuda.stream(st["d2h"]):
            dst[r0:r0 + m].copy_(buf, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st["d2h"])
            st["free"][k] = ev
    st["d2h"].synchronize()
    return out


def fft2(images, backend: CudaBackend | None = None):
    """2-D forward FFT of (..., rows, cols) complex64 (rows then columns)."""
    shape = tuple(images.shape)
    if len(shape) < 2:
        raise ValueError("fft2 needs at least 2 dimensions")
    rows, cols = shape[-2], shape[-1]
    stream, dev = _as_stream(images, rows * cols)
    backend = _backend_for(backend, dev)
    out = run(backend, fft2d_program(rows, cols), {"0.x": stream})["0.y"]
    return _unstream(out, shape, isinstance(out, DeviceStream))


# ---------------------------------------------------------------------------
# benchmark helpers (fft.py:180-262)

@dataclass(frozen=True)
class BenchRow:
    nbytes: int
    k: int
    seconds: float
    backend: str

    def csv(self) -> str:
        return f"{self.nbytes},{self.k},{self.seconds:.6f},{self.backend}"


def fft_bench(sizes: list[int], ks=(1, 2, 3), *, backend: CudaBackend | None = None,
              seed: int = 1234, warmup: bool = True, repeats: int = 1) -> list[BenchRow]:
    """Leaf-DFT streams of the given byte sizes through the device engine.

    As in the reference, only the engine is timed (plans built once); here
    the stream is device-resident and timed with CUDA events."""
    import torch

    from ..executor import chunk_arrays, plan, run_stream
    backend = backend or CudaBackend()
    rng = np.random.default_rng(seed)
    rows: list[BenchRow] = []
    for k in ks:
        width = 2 ** (k + 1)
        prog = leaf_program(k)
        p = plan(prog, backend.chunk_size, device=backend.device)
        if warmup:
            vals = torch.from_numpy(rng.standard_normal(width * 16, dtype=np.float32)).cuda()
            run_stream(p, chunk_arrays(p, {"0.x": vals}), writer=lambda c: None)
        for nbytes in sizes:
            items = max(1, nbytes // (4 * width))
            vals = torch.from_numpy(rng.standard_normal(items * width, dtype=np.float32)).cuda()
            best = float("inf")
            for _ in range(max(1, repeats)):
                start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                start.record()
                run_stream(p, chunk_arrays(p, {"0.x": vals}), writer=lambda c: None)
                stop.record()
                stop.synchronize()
                best = min(best, start.elapsed_time(stop) / 1e3)
            rows.append(BenchRow(items * width * 4, k, best, "b200"))
    return rows


def parse_sizes(spec: str) -> list[int]:
    """``"20K..10M"`` doubling ladder or ``"64K,1M"`` list (fft.py:241-262)."""
    def one(text: str) -> int:
        text = text.strip().upper()
        mult = {"K": 1024, "M": 1024 * 1024}.get(text[-1:], 1)
        return int(float(text[:-1] if mult > 1 else text) * mult)

    if ".." in spec:
        lo, hi = (one(t) for t in spec.split("..", 1))
        sizes = []
        while lo < hi:
            sizes.append(lo)
            lo *= 2
        return sizes + [hi]
    return [one(part) for part in spec.split(",")]

