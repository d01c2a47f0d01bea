"""Native execution of arbitrary kernel-language nodes.

A node whose body matches no hand-written implementation (nodes.py) is
parsed and type-checked (kernel/), translated to CUDA C (kernel/codegen.py)
and compiled once per (body, io) with NVRTC for sm_100a through the C ABI
(dpp_jit_compile).  ``JitNode.launch`` runs one thread per work-item on the
executor's stream, with the reference engine's contract (engine.py:193-195,
218-235): outputs start zero-filled, a bounds / division / budget fault
raises ``KernelRuntimeError`` naming the work-item the lockstep interpreter
would report (earliest statement, then lowest work-item; recovered by
re-running that one work-item with the detail slot enabled).
"""

from __future__ import annotations

import ctypes as C
import hashlib
import threading

import torch

from . import _lib
from ._torch import stream_handle
from .errors import KernelError, KernelRuntimeError, PlanError
from .kernel import compile_kernel
from .kernel.codegen import FAULT_BUDGET, FAULT_DIV, FAULT_INDEX, FAULT_MOD, generate
from .nodes import NativeNode, _io_of

__all__ = ["JitNode", "jit_node"]

_cache: dict[str, "JitNode"] = {}
_lock = threading.Lock()


class JitNode(NativeNode):
    def __init__(self, node, budget: int = 10_000_000):
        super().__init__(f"jit:{node.name}", _io_of(node))
        try:
            self.typed = compile_kernel(node.body, {p.name: p for p in node.io})
        except KernelError as exc:
            raise PlanError(f"kernel {node.name!r}: {exc}") from exc
        digest = hashlib.sha256((node.body + repr(sorted(self.io.items()))).encode()).hexdigest()[:16]
        self.fn = f"dpp_node_{digest}"
        self.source, self.params = generate(self.typed, self.fn, budget)
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

    def _launch(self, items, tensors, counts, gid0, fault, diag, stream):
        vals = [t.data_ptr() for t in tensors] + counts + [items, self.global_size, gid0, fault.data_ptr(),
                                                            0 if diag is None else diag.data_ptr()]
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
        key = int(fault.cpu().item()) & 0xFFFFFFFFFFFFFFFF  # synchronises the stream
        if key == 0xFFFFFFFFFFFFFFFF:
            return
        gid = key & 0xFFFFFFFF
        diag = torch.zeros(3, dtype=torch.int64, device=dev)
        fault2 = torch.full((1,), -1, dtype=torch.int64, device=dev)
        self._launch(1, tensors, counts, gid, fault2, diag, stream)
        code, pt, value = (int(v) for v in diag.cpu().tolist())
        if code == FAULT_INDEX:
            p = self.points[pt]
            msg = f"index {value} out of range for point {p.name!r} (0..{counts[pt] - 1})"
        elif code == FAULT_DIV:
            msg = "integer division by zero"
        elif code == FAULT_MOD:
            msg = "integer modulo by zero"
        elif code == FAULT_BUDGET:
            msg = "instruction budget exceeded"
        else:  # pragma: no cover
            msg = "kernel fault"
        raise KernelRuntimeError(msg, work_item=gid)


def jit_node(node) -> JitNode:
    """Compiled node for ``node`` (cached by body and io signature)."""
    key = node.body + "\x00" + repr(_io_of(node))
    with _lock:
        jn = _cache.get(key)
        if jn is None:
            jn = JitNode(node)
            _cache[key] = jn
    return jn
