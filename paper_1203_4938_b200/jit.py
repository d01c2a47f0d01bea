"""Native execution of arbitrary kernel-language nodes.

A node whose body matches no hand-written implementation (nodes.py) is
parsed and type-checked (kernel/), translated to CUDA C (kernel/codegen.py)
and compiled once per (body, io) with NVRTC for sm_100a through the C ABI
(dpp_jit_compile).  ``JitNode.launch`` runs one thread per work-item on the
executor's stream, with the reference engine's contract (engine.py:193-195,
218-235): outputs start zero-filled, a bounds / division / budget fault
raises ``KernelRuntimeError`` naming the work-item the lockstep interpreter
would report (the earliest fault in lockstep order, then the lowest
work-item; kernel/codegen.py).  Launches inside ``deferred_faults()`` (every
``client.run``) are not synchronised: their fault words are read once when
the run ends.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import threading

import torch

from . import _lib
from ._torch import stream_handle
from .errors import EngineRuntimeError, KernelError, KernelRuntimeError, PlanError
from .kernel import compile_kernel
from .kernel.codegen import FAULT_BUDGET, FAULT_DIV, FAULT_INDEX, FAULT_MOD, generate
from .nodes import NativeNode, _io_of

__all__ = ["JitNode", "jit_node", "deferred_faults", "set_site"]

_cache: dict[str, "JitNode"] = {}
_lock = threading.Lock()


_scope = threading.local()


class deferred_faults:
    """Collect the fault words of every JIT launch inside the scope and check
    them once, at exit, with one host synchronisation (client.run wraps a
    whole run in it) instead of one per launch.  The first faulting launch in
    launch order is diagnosed and raised as ``EngineRuntimeError`` with its
    instance and chunk (engine.py:199-205)."""

    def __enter__(self):
        self.prev = getattr(_scope, "records", None)
        _scope.records = []
        return self

    def __exit__(self, exc_type, exc, tb):
        records, _scope.records = _scope.records, self.prev
        if exc_type is not None or not records:
            return False
        words = torch.stack([r[0].fault for r in records]).cpu()  # the one synchronisation
        for (rec, iid, chunk), w in zip(records, words.tolist()):
            if w[0] != -1:
                try:
                    rec.raise_fault()
                except KernelRuntimeError as err:
                    raise EngineRuntimeError(str(err), instance=iid, work_item=err.work_item,
                                             chunk=chunk) from err
        return False


def set_site(iid, chunk) -> None:
    """The executor names the instance and chunk of the launches that follow."""
    _scope.site = (iid, chunk)


class _Launch:
    """One launch of a JIT node: enough to re-run it for the fault diagnosis."""

    def __init__(self, node, items, tensors, counts, fault, stream):
        self.node, self.items, self.tensors, self.counts = node, items, tensors, counts
        self.fault, self.stream = fault, stream

    def raise_fault(self):
        """Re-run the node to find the fault the lockstep evaluator reports
        first: the minimum (loop region, iteration, ..., site) tuple, one
        component per pass, then the lowest work-item, then its detail."""
        node, dev = self.node, self.fault.device
        prefix: list[int] = []
        pbuf = torch.zeros(64, dtype=torch.int64, device=dev)
        while True:
            m = len(prefix)
            if m:
                pbuf[:m] = torch.tensor(prefix, dtype=torch.int64)
            f = torch.full((1,), -1, dtype=torch.int64, device=dev)
            node._launch(self.items, self.tensors, self.counts, 0, f, None, self.stream, m, pbuf.data_ptr())
            v = int(f.item())
            if v < 0 or m >= 63:  # pragma: no cover (a normal launch flagged this fault)
                raise KernelRuntimeError("kernel fault")
            prefix.append(v)
            if m % 2 == 0 and v in node.sites:  # regions and sites sit at even positions
                break
        f = torch.full((1,), -1, dtype=torch.int64, device=dev)
        pbuf[:len(prefix)] = torch.tensor(prefix, dtype=torch.int64)
        node._launch(self.items, self.tensors, self.counts, 0, f, None, self.stream, len(prefix), pbuf.data_ptr())
        gid = int(f.item())
        diag = torch.zeros(3, dtype=torch.int64, device=dev)
        f = torch.full((1,), -1, dtype=torch.int64, device=dev)
        node._launch(1, self.tensors, self.counts, gid, f, diag, self.stream)
        code, pt, value = (int(v) for v in diag.cpu().tolist())
        if code == FAULT_INDEX:
            p = node.points[pt]
            msg = f"index {value} out of range for point {p.name!r} (0..{self.counts[pt] - 1})"
        elif code == FAULT_DIV:
            msg = "integer division by zero"
        elif code == FAULT_MOD:
            msg = "integer modulo by zero"
        elif code == FAULT_BUDGET:
            raise KernelRuntimeError("instruction budget exceeded")  # no work-item (interp.py:124-126)
        else:  # pragma: no cover
            msg = "kernel fault"
        raise KernelRuntimeError(msg, work_item=gid)


class JitNode(NativeNode):
    def __init__(self, node, budget: int = 10_000_000):
        super().__init__(f"jit:{node.name}", _io_of(node))
        try:
            self.typed = compile_kernel(node.body, {p.name: p for p in node.io})
        except KernelError as exc:
            raise PlanError(f"kernel {node.name!r}: {exc}") from exc
        digest = hashlib.sha256((node.body + repr(sorted(self.io.items()))).encode()).hexdigest()[:16]
        self.fn = f"dpp_node_{digest}"
        self.source, self.params, self.sites = generate(self.typed, self.fn, budget)
        self.points = list(self.typed.io.values())
        lib = _lib.load()
        h = C.c_void_p()
        log = C.create_string_buffer(8192)
        _lib.check(lib.dpp_jit_compile(self.source.encode(), self.fn.encode(), C.byref(h), log, len(log)),
                   f"kernel {node.name!r}")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().dpp_jit_destroy(h)
            except Exception:  # interpreter shutdown
                pass

    def _launch(self, items, tensors, counts, gid0, fault, diag, stream, mode=-1, prefix=0):
        vals = [t.data_ptr() for t in tensors] + counts + [items, self.global_size, gid0, fault.data_ptr(),
                                                            0 if diag is None else diag.data_ptr(), mode, prefix]
        arr = (C.c_uint64 * len(vals))(*[v & 0xFFFFFFFFFFFFFFFF for v in vals])
        _lib.check(_lib.load().dpp_jit_launch(self._h, arr, len(vals), items, stream_handle(stream)),
                   f"kernel {self.kind}")

    def launch(self, items, inputs, outputs, stream):
        dev = next(iter(outputs.values())).device if outputs else next(iter(inputs.values())).device
        for t in outputs.values():
            t.zero_()  # the reference engine hands zero-filled outputs (engine.py:193-195)
        tensors = [inputs[p.name] if p.is_input else outputs[p.name] for p in self.points]
        counts = [t.numel() // p.data.width for t, p in zip(tensors, self.points)]
        self.global_size = items
        fault = torch.full((1,), -1, dtype=torch.int64, device=dev)
        self._launch(items, tensors, counts, 0, fault, None, stream)
        rec = _Launch(self, items, tensors, counts, fault, stream)
        records = getattr(_scope, "records", None)
        if records is not None:  # checked once at the end of the run
            iid, chunk = getattr(_scope, "site", (None, None))
            records.append((rec, iid, chunk))
            return
        if int(fault.cpu().item()) != -1:  # direct call: check now
            rec.raise_fault()


def jit_node(node) -> JitNode:
    """Compiled node for ``node`` (cached by body and io signature)."""
    key = node.body + "\x00" + repr(_io_of(node))
    with _lock:
        jn = _cache.get(key)
        if jn is None:
            jn = JitNode(node)
            _cache[key] = jn
    return jn
