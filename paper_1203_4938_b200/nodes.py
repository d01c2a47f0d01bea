"""Native-node registry: binds graph kernels to sm_100a implementations.

The reference executes every node by interpreting its body
(engine.py:218-235 -> interp.run_lanes).  This framework instead matches
each kernel against the registered native implementations by
(name, io signature, exact body text) — the bodies are the ones the
reference's own program builders generate (apps/fft.py:86-123,
apps/imgc.py:128-185) plus this framework's self-describing whole-transform
and fused-codec nodes — and compiles any other body to sm_100a with NVRTC (``jit.py``); bodies that
do not parse or type-check are a ``PlanError``.  There is no interpreter and
no CPU fallback.

Each ``NativeNode.launch`` receives flat device tensors exactly as the
reference's ``_run_instance`` receives flat numpy buffers (item count, inputs
by point name, outputs pre-allocated by the executor) and enqueues kernels on
the given stream.
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field

import torch

from . import ops
from .errors import KernelRuntimeError, PlanError
from .types import DataType, Direction

__all__ = ["NativeNode", "resolve", "register", "registered_kinds"]


@dataclass
class NativeNode:
    kind: str
    io: dict[str, tuple[str, int, str]]  # point -> (base, width, direction)
    broadcast: frozenset = field(default_factory=frozenset)  # inputs not chunked (side inputs)
    # points whose element count differs from the work-item count: point -> (num, den)
    ratio: dict = field(default_factory=dict)

    def check_items(self, items: int) -> None:
        """Raise KernelRuntimeError if the chunk cannot be executed (reference-style fault)."""

    def launch(self, items: int, inputs: dict, outputs: dict, stream) -> None:  # pragma: no cover
        raise NotImplementedError


def _io_of(node) -> dict[str, tuple[str, int, str]]:
    return {p.name: (p.data.base, p.data.width, p.direction.value) for p in node.io}


_IN, _OUT = Direction.INPUT.value, Direction.OUTPUT.value


# ---------------------------------------------------------------------------
# FFT nodes

class LeafNode(NativeNode):
    """dft{2,4,8} (apps/fft.py:86-117): bit-exact native evaluation."""

    def __init__(self, k: int):
        w = 2 << k
        super().__init__(f"dft{1 << k}", {"x": ("float", w, _IN), "y": ("float", w, _OUT)})
        self.k = k

    def launch(self, items, inputs, outputs, stream):
        ops.leaf_dft(self.k, inputs["x"], outputs["y"], stream)


class FftNode(NativeNode):
    """fft{n}: whole forward transforms over runs of n work-items."""

    def __init__(self, n: int):
        super().__init__(f"fft{n}", {"x": ("float", 2, _IN), "y": ("float", 2, _OUT)})
        self.n = n

    def check_items(self, items):
        if items % self.n:
            base = items - items % self.n
            raise KernelRuntimeError(f"index {items} out of range for point 'x' (0..{items - 1})",
                                     work_item=base)

    def launch(self, items, inputs, outputs, stream):
        x = torch.view_as_complex(inputs["x"].view(-1, 2))
        y = torch.view_as_complex(outputs["y"].view(-1, 2))
        ops.fft_forward(x, self.n, out=y, stream=stream)


class Fft2dNode(NativeNode):
    """fft2d_{r}x{c}: whole 2-D transforms over runs of r*c work-items."""

    def __init__(self, rows: int, cols: int):
        super().__init__(f"fft2d_{rows}x{cols}", {"x": ("float", 2, _IN), "y": ("float", 2, _OUT)})
        self.rows, self.cols = rows, cols

    def check_items(self, items):
        size = self.rows * self.cols
        if items % size:
            raise KernelRuntimeError(f"index {items} out of range for point 'x' (0..{items - 1})",
                                     work_item=items - items % size)

    def launch(self, items, inputs, outputs, stream):
        x = torch.view_as_complex(inputs["x"].view(-1, 2))
        y = torch.view_as_complex(outputs["y"].view(-1, 2))
        ops.fft2d_forward(x, self.rows, self.cols, out=y, stream=stream)


# ---------------------------------------------------------------------------
# codec nodes (apps/imgc.py:128-185)

class YccNode(NativeNode):
    def __init__(self):
        super().__init__("ycbcr", {"rgb": ("uchar", 4, _IN), "yl": ("float", 1, _OUT),
                                   "cb": ("float", 1, _OUT), "cr": ("float", 1, _OUT)})

    def launch(self, items, inputs, outputs, stream):
        ops.ycbcr(inputs["rgb"], outputs["yl"], outputs["cb"], outputs["cr"], stream)


class BoxdownNode(NativeNode):
    def __init__(self):
        super().__init__("boxdown", {"blk": ("float", 16, _IN), "avg": ("float", 1, _OUT)})

    def launch(self, items, inputs, outputs, stream):
        ops.boxdown(inputs["blk"], outputs["avg"], stream)


class GradientNode(NativeNode):
    def __init__(self, width: int, height: int):
        super().__init__("gradient", {"lum": ("float", 1, _IN), "dx": ("float", 1, _OUT),
                                      "dy": ("float", 1, _OUT)})
        self.width, self.height = width, height

    def launch(self, items, inputs, outputs, stream):
        ops.gradient(inputs["lum"], outputs["dx"], outputs["dy"], self.width, self.height, stream)


class VqNode(NativeNode):
    def __init__(self, size: int):
        super().__init__("vqnearest", {"blk": ("float", 16, _IN), "cbk": ("float", 16, _IN),
                                       "idx": ("int", 1, _OUT)})
        self.size = size

    def launch(self, items, inputs, outputs, stream):
        ops.vqnearest(inputs["blk"], inputs["cbk"], outputs["idx"], self.size, stream)


class EncodeNode(NativeNode):
    """Fused codec node ``imgc_encode`` (this framework's extension).

    io: px uchar16 (16 consecutive raster gray pixels per work-item, so one
    work-item per 4x4 block), cbk float16 (broadcast side input: the
    codebook, not chunked), outputs mu/sig/idx/cb/cr uchar per block in
    raster block order.  Frame geometry is baked into the body like the
    reference's gradient node (imgc.py:155-166)."""

    def __init__(self, width: int, height: int, ncb: int):
        super().__init__("imgc_encode",
                         {"px": ("uchar", 16, _IN), "cbk": ("float", 16, _IN),
                          **{p: ("uchar", 1, _OUT) for p in ("mu", "sig", "idx", "cb", "cr")}},
                         broadcast=frozenset({"cbk"}))
        self.width, self.height, self.ncb = width, height, ncb
        self.blocks = (width // 4) * (height // 4)

    def check_items(self, items):
        if items % self.blocks:
            raise KernelRuntimeError(f"chunk of {items} blocks is not a whole number of "
                                     f"{self.width}x{self.height} frames",
                                     work_item=items - items % self.blocks)

    def launch(self, items, inputs, outputs, stream):
        batch = items // self.blocks
        cbk = inputs["cbk"]
        shared = cbk.numel() == self.ncb * 16
        if not shared and cbk.numel() != self.ncb * 16 * batch:
            raise KernelRuntimeError(f"codebook stream holds {cbk.numel() // 16} centroids, node expects "
                                     f"{self.ncb} (shared) or {self.ncb} per frame", work_item=0)
        # the record bytes land directly in the mu / sig / idx output planes
        ops.encode_planar(inputs["px"], self.height, self.width, cbk, outputs["mu"], outputs["sig"],
                          outputs["idx"], outputs["cb"], outputs["cr"], batch=batch,
                          shared_codebook=shared, stream=stream)


class ToComplexNode(NativeNode):
    """C5 adapter: gray u8 -> complex64 (g, 0) (apps/chain.py)."""

    def __init__(self):
        super().__init__("to_complex", {"x": ("uchar", 1, _IN), "y": ("float", 2, _OUT)})

    def launch(self, items, inputs, outputs, stream):
        ops.u8_to_complex(inputs["x"], outputs["y"], stream)


class SpectrumU8Node(NativeNode):
    """C5 adapter: complex64 -> u8 clip(floor(alpha*log(1+|z|))) (apps/chain.py)."""

    def __init__(self, alpha: float):
        super().__init__("spectrum_u8", {"x": ("float", 2, _IN), "y": ("uchar", 1, _OUT)})
        self.alpha = alpha

    def launch(self, items, inputs, outputs, stream):
        ops.spectrum_u8(inputs["x"], outputs["y"], self.alpha, stream)


# ---------------------------------------------------------------------------
# registry

_MATCHERS = []


def register(matcher):
    """Add ``matcher(node) -> NativeNode | None`` to the registry."""
    _MATCHERS.append(matcher)
    return matcher


def registered_kinds() -> list[str]:
    return [m.__name__ for m in _MATCHERS]


def _same_io(native: NativeNode, node) -> bool:
    return native.io == _io_of(node)


@register
def match_leaf(node):
    from .apps.fft import leaf_kernel
    for k in (1, 2, 3):
        if node.body == leaf_kernel(k).body:
            return LeafNode(k)
    return None


@register
def match_fft(node):
    from .apps.fft import NATIVE_TAG, fft2d_kernel, fft_kernel
    m = re.match(re.escape(NATIVE_TAG) + r" fft n=(\d+)\n", node.body)
    if m:
        n = int(m.group(1))
        return FftNode(n) if node.body == fft_kernel(n).body else None
    m = re.match(re.escape(NATIVE_TAG) + r" fft2d rows=(\d+) cols=(\d+)\n", node.body)
    if m:
        r, c = int(m.group(1)), int(m.group(2))
        if node.body != fft2d_kernel(r, c).body:
            return None
        # shapes without a native 2-D schedule (column length < 256, or rows
        # narrower than a column tile) run the node's own naive-DFT body
        # through the JIT: the document's meaning, on the GPU, just O(N^2)
        from . import ops
        return Fft2dNode(r, c) if ops.fft_shape_supported(2, r, c) else None
    return None


@register
def match_codec(node):
    from .apps import imgc
    if node.body == imgc.ycbcr_program().kernels["ycbcr"].body:
        return YccNode()
    if node.body == imgc.chroma_down_program().kernels["boxdown"].body:
        return BoxdownNode()
    m = re.search(r"int x = i % (\d+);\nint y = i / \1;", node.body)
    if m:
        w = int(m.group(1))
        mh = re.search(r"\(y < (\d+)\)", node.body)
        if mh:
            h = int(mh.group(1)) + 1
            if node.body == imgc.gradient_program(w, h).kernels["gradient"].body:
                return GradientNode(w, h)
    m = re.search(r"for \(int j = 0; j < (\d+); j = j \+ 1\)", node.body)
    if m and node.name == "vqnearest":
        n = int(m.group(1))
        if node.body == imgc.vq_program(n).kernels["vqnearest"].body:
            return VqNode(n)
    m = re.match(re.escape(imgc.NATIVE_TAG) + r" imgc_encode width=(\d+) height=(\d+) ncb=(\d+)\n",
                 node.body)
    if m:
        w, h, n = map(int, m.groups())
        if node.body == imgc.encode_kernel(w, h, n).body:
            return EncodeNode(w, h, n)
    return None


@register
def match_chain(node):
    from .apps import chain
    if node.body == chain.to_complex_kernel().body:
        return ToComplexNode()
    m = re.search(r"float v = floor\(([0-9.e+-]+)f \* log\(1\.0f \+ m\)\);", node.body)
    if m:
        alpha = float(m.group(1))
        if node.body == chain.spectrum_u8_kernel(alpha).body:
            return SpectrumU8Node(alpha)
    return None


def resolve(node) -> NativeNode:
    """The native implementation of ``node`` or PlanError."""
    for matcher in _MATCHERS:
        native = matcher(node)
        if native is not None:
            if not _same_io(native, node):
                raise PlanError(f"kernel {node.name!r}: io {_io_of(node)} does not match the native "
                                f"{native.kind} signature {native.io}")
            return native
    # no hand-written kernel: compile the body itself for sm_100a (NVRTC);
    # parse / type errors surface as PlanError like the reference's plan()
    from .jit import jit_node
    return jit_node(node)


_ = DataType
