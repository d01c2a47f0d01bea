"""Device executor: the reference engine's plan/chunk/run contract on CUDA streams.

Mirrors /root/reference/pkg/src/dpp/engine.py with the same names and rules:

* ``plan`` (engine.py:82-135): structural validation, topological order,
  width-conversion multipliers as ``Fraction`` (engine.py:108-109), input
  bindings ``("free", stream)`` / ``("arrow", iid, point)``; kernel bodies are
  bound to native implementations (``nodes.resolve``) instead of compiled.
  Plans are cached by (program id, chunk size, device) — the reference
  recompiles on every call (~7 ms per ``fft()``).
* ``chunk_arrays`` (engine.py:397-424): W-element chunks as tensor VIEWS.
* ``run_chunk`` (engine.py:176-215): every instance in topological order;
  outputs allocated on the device; producer buffers handed to consumers by
  reference, so edges never leave HBM.
* ``run_stream`` (engine.py:255-330): ordered emission; chunks are enqueued
  back to back on one CUDA stream (stream order replaces the thread pool;
  ``pool="process"`` is refused because CUDA contexts do not survive fork).

Extension: a native node may declare *broadcast* inputs
(side inputs such as a codebook) that are handed whole to every chunk and
excluded from the equal-element-count rule.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Callable, Iterable, Iterator

import torch

from .errors import EngineRuntimeError, KernelRuntimeError, PlanError
from .model import FreePoint, Program, as_program, free_points, program_id, topological_order, validate
from .nodes import NativeNode, resolve
from .types import Direction
from ._torch import nvtx_range, require_cuda, torch_dtype

__all__ = ["DEFAULT_CHUNK_SIZE", "ExecutionPlan", "Chunk", "RunResult", "plan", "run_chunk",
           "run_stream", "chunk_arrays"]

DEFAULT_CHUNK_SIZE = None  # whole stream in one chunk (the reference default is 4096)


@dataclass(frozen=True)
class ExecutionPlan:
    program: Program
    order: tuple[int, ...]
    multipliers: dict[int, Fraction]
    kernels: dict[str, NativeNode]
    bindings: dict[tuple[int, str], tuple]
    free_inputs: tuple[FreePoint, ...]
    free_outputs: tuple[FreePoint, ...]
    chunk_size: int | None
    device: torch.device
    broadcast: frozenset = frozenset()  # free input stream names handed whole to every chunk
    # fusion: fft2d instance -> (to_complex instance, spectrum_u8 instance) run as one
    # fused launch (ops.fft2d_u8_spectrum); the two adapters are then skipped
    fused: dict = field(default_factory=dict)
    absorbed: frozenset = frozenset()

    @property
    def items_per_element(self) -> Fraction:
        return sum(self.multipliers.values(), Fraction(0))

    @property
    def counted_inputs(self) -> tuple[FreePoint, ...]:
        return tuple(fp for fp in self.free_inputs if fp.stream not in self.broadcast)


@dataclass
class Chunk:
    """One block of stream data: flat device (or host) buffers keyed by stream name."""

    index: int
    buffers: dict[str, object]
    counts: dict[str, int]


@dataclass
class RunResult:
    chunks: list[Chunk] = field(default_factory=list)
    total_work_items: int = 0
    events: list = field(default_factory=list, repr=False)

    @property
    def timings(self) -> list[float]:
        """Per-chunk device seconds (engine.py:65-69); waits for the stream on first use."""
        if self.events:
            self.events[-1][1].synchronize()
        return [a.elapsed_time(b) / 1e3 for a, b in self.events]


_cache: dict[tuple, ExecutionPlan] = {}
_cache_lock = threading.Lock()


def plan(program, chunk_size: int | None = DEFAULT_CHUNK_SIZE, *, device=None) -> ExecutionPlan:
    """Validate, bind native nodes and fix the schedule (engine.py:82-135)."""
    if chunk_size is not None and chunk_size < 1:
        raise PlanError(f"chunk size must be >= 1, got {chunk_size}")
    program = as_program(program)
    dev = require_cuda(device)
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (program_id(program), chunk_size, dev.index)
    with _cache_lock:
        hit = _cache.get(key)
    if hit is not None:
        return hit
    report = validate(program)
    if not report.ok:
        raise PlanError(f"program is not executable:\n{report}")
    kernels = {name: resolve(node) for name, node in program.kernels.items()}
    order = tuple(topological_order(program))
    producers = {a.input: a.output for a in program.arrows}
    bindings: dict[tuple[int, str], tuple] = {}
    multipliers: dict[int, Fraction] = {}
    broadcast: set[str] = set()
    for iid in order:
        inst = program.instance(iid)
        node = program.kernels[inst.kernel]
        native = kernels[inst.kernel]
        cands: list[tuple[str, Fraction]] = []
        for p in node.io:
            if not p.is_input:
                continue
            key_p = (iid, p.name)
            if key_p in producers:
                src = producers[key_p]
                if p.name in native.broadcast:
                    raise PlanError(f"broadcast input {iid}.{p.name} must be a free stream")
                m = multipliers[src[0]] * program.point_of(*src).data.width / p.data.width
                bindings[key_p] = ("arrow", src[0], src[1])
            else:
                m = Fraction(1)
                bindings[key_p] = ("free", f"{iid}.{p.name}")
                if p.name in native.broadcast:
                    broadcast.add(f"{iid}.{p.name}")
                    continue
            cands.append((p.name, m))
        first = cands[0][1]
        for pname, m in cands[1:]:
            if m != first:
                raise PlanError(f"work-item count mismatch at instance {iid}: point {cands[0][0]!r} "
                                f"implies x{first}, {pname!r} implies x{m}")
        if chunk_size is not None and (first * chunk_size).denominator != 1:
            raise PlanError(f"non-integral width conversion: instance {iid} runs {first} work-items per "
                            f"element, not integral at chunk size {chunk_size}")
        multipliers[iid] = first
    free = free_points(program)
    fused = _fusions(program, kernels, bindings, free, multipliers)
    result = ExecutionPlan(
        program=program, order=order, multipliers=multipliers, kernels=kernels, bindings=bindings,
        free_inputs=tuple(p for p in free if p.direction is Direction.INPUT),
        free_outputs=tuple(p for p in free if p.direction is Direction.OUTPUT),
        chunk_size=chunk_size, device=dev, broadcast=frozenset(broadcast), fused=fused,
        absorbed=frozenset(i for pair in fused.values() for i in pair))
    with _cache_lock:
        _cache[key] = result
    return result


def _fusions(program, kernels, bindings, free, multipliers) -> dict:
    """to_complex -> fft2d_RxC -> spectrum_u8 chains whose intermediate edges have
    no other consumer (and are not free outputs) -> {fft2d iid: (tc iid, spec iid)}.
    Only shapes with a fused schedule (4096 columns, ring column pass) qualify;
    DPP_FUSE=0 disables the pass."""
    import os
    if os.environ.get("DPP_FUSE") == "0":
        return {}
    consumers: dict = {}
    for a in program.arrows:
        consumers.setdefault(a.output, []).append(a.input)
    free_out = {(fp.instance, fp.point) for fp in free if fp.direction is Direction.OUTPUT}
    kind = {inst.id: kernels[inst.kernel].kind for inst in program.nodes}
    out = {}
    for inst in program.nodes:
        native = kernels[inst.kernel]
        if not native.kind.startswith("fft2d_") or getattr(native, "cols", None) != 4096 or \
                native.rows not in (4096, 16384):
            continue
        src = bindings.get((inst.id, "x"))
        if src is None or src[0] != "arrow" or kind.get(src[1]) != "to_complex":
            continue
        tc = src[1]
        if consumers.get((tc, "y"), []) != [(inst.id, "x")] or (tc, "y") in free_out:
            continue
        outs = consumers.get((inst.id, "y"), [])
        if len(outs) != 1 or (inst.id, "y") in free_out or kind.get(outs[0][0]) != "spectrum_u8":
            continue
        sp = outs[0][0]
        if multipliers[tc] != multipliers[inst.id] or multipliers[sp] != multipliers[inst.id]:
            continue
        out[inst.id] = (tc, sp)
    return out


def _element_count(p: ExecutionPlan, chunk: Chunk) -> int:
    counts = set()
    for fp in p.free_inputs:
        if fp.stream not in chunk.buffers:
            raise EngineRuntimeError(f"missing input stream {fp.stream!r}", chunk=chunk.index)
        if fp.stream in p.broadcast:
            continue
        buf = chunk.buffers[fp.stream]
        n = buf.numel()
        count = chunk.counts.get(fp.stream, n // fp.data.width)
        if buf.dtype != torch_dtype(fp.data):
            raise EngineRuntimeError(f"stream {fp.stream!r} carries {buf.dtype}, expected {fp.data}",
                                     chunk=chunk.index)
        if n != count * fp.data.width:
            raise EngineRuntimeError(f"stream {fp.stream!r}: buffer holds {n} scalars, expected "
                                     f"{count * fp.data.width}", chunk=chunk.index)
        counts.add(count)
    unknown = chunk.buffers.keys() - {fp.stream for fp in p.free_inputs}
    if unknown:
        raise EngineRuntimeError(f"unexpected input stream {sorted(unknown)[0]!r}", chunk=chunk.index)
    if len(counts) > 1:
        raise EngineRuntimeError(f"input streams disagree on element count: {sorted(counts)}",
                                 chunk=chunk.index)
    return counts.pop() if counts else 0


def _jit():
    from . import jit
    return jit


def _items(p: ExecutionPlan, iid: int, elements: int, chunk_index: int) -> int:
    items = p.multipliers[iid] * elements
    if items.denominator != 1:
        raise EngineRuntimeError(f"width conversion not integral for instance {iid} at {elements} "
                                 f"elements", chunk=chunk_index)
    return int(items)


def _run_one(p: ExecutionPlan, iid: int, chunk: Chunk, elements: int, produced: dict, stream) -> None:
    inst = p.program.instance(iid)
    node = p.program.kernels[inst.kernel]
    native = p.kernels[inst.kernel]
    items = _items(p, iid, elements, chunk.index)
    inputs = {}
    for pt in node.io:
        if not pt.is_input:
            continue
        kind = p.bindings[(iid, pt.name)]
        inputs[pt.name] = chunk.buffers[kind[1]] if kind[0] == "free" else produced[(kind[1], kind[2])]
    outputs = {pt.name: torch.empty(items * pt.data.width, dtype=torch_dtype(pt.data), device=p.device)
               for pt in node.io if not pt.is_input}
    try:
        if items:
            native.check_items(items)
            _jit().set_site(iid, chunk.index)
            with nvtx_range(f"{native.kind}[{iid}]"):
                native.launch(items, inputs, outputs, stream)
    except KernelRuntimeError as exc:
        raise EngineRuntimeError(str(exc), instance=iid, work_item=exc.work_item,
                                 chunk=chunk.index) from exc
    for name, buf in outputs.items():
        produced[(iid, name)] = buf


def run_chunk(p: ExecutionPlan, chunk: Chunk, stream: torch.cuda.Stream | None = None) -> Chunk:
    """Run every instance over one chunk on ``stream`` (engine.py:176-215)."""
    elements = _element_count(p, chunk)
    produced: dict[tuple[int, str], torch.Tensor] = {}
    for iid in p.order:
        if iid in p.absorbed:
            continue
        if iid in p.fused:
            if not _run_fused(p, iid, chunk, elements, produced, stream):
                tc, sp = p.fused[iid]
                for j in (tc, iid, sp):  # no fused schedule after all: the three nodes
                    _run_one(p, j, chunk, elements, produced, stream)
            continue
        _run_one(p, iid, chunk, elements, produced, stream)
    out_buf, out_cnt = {}, {}
    for fp in p.free_outputs:
        out_buf[fp.stream] = produced[(fp.instance, fp.point)]
        out_cnt[fp.stream] = _items(p, fp.instance, elements, chunk.index)
    return Chunk(chunk.index, out_buf, out_cnt)


def _run_fused(p: ExecutionPlan, iid: int, chunk: Chunk, elements: int, produced: dict, stream) -> bool:
    """to_complex -> fft2d -> spectrum_u8 as one fused launch (False: not possible
    for this chunk; the caller then runs the three instances one by one)."""
    from . import ops
    tc, sp = p.fused[iid]
    native = p.kernels[p.program.instance(iid).kernel]
    items = _items(p, iid, elements, chunk.index)
    kind = p.bindings[(tc, "x")]
    x = chunk.buffers[kind[1]] if kind[0] == "free" else produced[(kind[1], kind[2])]
    try:
        native.check_items(items)
    except KernelRuntimeError as exc:
        raise EngineRuntimeError(str(exc), instance=iid, work_item=exc.work_item, chunk=chunk.index) from exc
    y = torch.empty(items, dtype=torch.uint8, device=p.device)
    alpha = p.kernels[p.program.instance(sp).kernel].alpha
    if items and not ops.fft2d_u8_spectrum(x, native.rows, native.cols, alpha, y, stream):
        return False
    produced[(sp, "y")] = y
    return True


def _checked(p: ExecutionPlan, chunks: Iterable[Chunk]) -> Iterator[tuple[int, Chunk, int]]:
    """Dense indices, short chunk only last (engine.py:339-361)."""
    expected, short = 0, None
    for chunk in chunks:
        if chunk.index != expected:
            raise EngineRuntimeError(f"chunk {chunk.index} arrived out of order (expected {expected})",
                                     chunk=chunk.index)
        if short is not None:
            raise EngineRuntimeError(f"short chunk {short} was not the final chunk", chunk=chunk.index)
        elements = _element_count(p, chunk)
        if p.chunk_size is not None:
            if elements > p.chunk_size:
                raise EngineRuntimeError(f"chunk carries {elements} elements, plan chunk size is "
                                         f"{p.chunk_size}", chunk=chunk.index)
            if elements < p.chunk_size:
                short = chunk.index
        yield chunk.index, chunk, elements
        expected += 1


def run_stream(p: ExecutionPlan, chunks: Iterable[Chunk], writer: Callable[[Chunk], None] | None = None,
               *, workers: int = 1, max_in_flight: int | None = None, pool: str = "thread",
               stream: torch.cuda.Stream | None = None) -> RunResult:
    """Whole stream, outputs emitted in input order (engine.py:255-330).

    Chunks are enqueued back to back on ``stream`` without host syncs;
    ``RunResult.timings`` reads the per-chunk CUDA events when asked."""
    if pool not in ("thread", "process"):
        raise ValueError(f"unknown pool kind {pool!r}")
    if pool == "process" and workers > 1:
        raise PlanError("pool='process' is not supported by the device engine (CUDA does not survive "
                        "fork); chunks are pipelined on CUDA streams instead")
    result = RunResult()
    per_element = p.items_per_element
    s = stream if stream is not None else torch.cuda.current_stream(p.device)
    with torch.cuda.device(p.device):
        for _, chunk, elements in _checked(p, chunks):
            start = torch.cuda.Event(enable_timing=True)
            stop = torch.cuda.Event(enable_timing=True)
            start.record(s)
            with nvtx_range(f"chunk {chunk.index}"):
                out = run_chunk(p, chunk, s)
            stop.record(s)
            result.events.append((start, stop))
            result.total_work_items += int(per_element * elements)
            if writer is not None:
                writer(out)
            else:
                result.chunks.append(out)
    return result


def chunk_arrays(p: ExecutionPlan, streams: dict[str, object]) -> Iterator[Chunk]:
    """Cut whole device streams into plan-sized chunks of views (engine.py:397-424)."""
    counts = set()
    for fp in p.free_inputs:
        if fp.stream not in streams:
            raise EngineRuntimeError(f"missing input stream {fp.stream!r}")
        if fp.stream not in p.broadcast:
            counts.add(streams[fp.stream].numel() // fp.data.width)
    extra = streams.keys() - {fp.stream for fp in p.free_inputs}
    if extra:
        raise EngineRuntimeError(f"unexpected input stream {sorted(extra)[0]!r}")
    if len(counts) > 1:
        raise EngineRuntimeError(f"input streams disagree on element count: {sorted(counts)}")
    total = counts.pop() if counts else 0
    w = p.chunk_size or max(total, 1)
    for index in range((total + w - 1) // w):
        lo, hi = index * w, min((index + 1) * w, total)
        bufs, cnts = {}, {}
        for fp in p.free_inputs:
            t = streams[fp.stream]
            if fp.stream in p.broadcast:
                bufs[fp.stream] = t
                continue
            bufs[fp.stream] = t[lo * fp.data.width:hi * fp.data.width]
            cnts[fp.stream] = hi - lo
        yield Chunk(index, bufs, cnts)
