"""``run(backend, program, inputs)`` on the B200 engine (mirror of dpp.client).

Same contract as /root/reference/pkg/src/dpp/client.py:77-104: one stream per
free input point keyed ``"<instance>.<point>"``, one returned per free output
point, the same ``ClientError`` checks (client.py:48-74).  Inputs may be host
``StreamFile`` objects (staged H2D through pinned memory) or device-resident
``DeviceStream`` objects; outputs come back as ``StreamFile`` (one D2H per free
output) unless ``CudaBackend(outputs="device")``.

``LocalBackend`` is kept as an alias so code written against the reference's
in-process backend runs unchanged — in-process here means the local GPU.
``RemoteBackend`` (HTTP/TCP server path) is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ClientError
from .model import as_program, free_points
from .types import Direction
from .wire import DeviceStream, StreamFile

__all__ = ["CudaBackend", "LocalBackend", "run"]


@dataclass(frozen=True)
class CudaBackend:
    """In-process execution on one CUDA device.

    chunk_size: work-items per chunk (None = whole stream; the reference's
      LocalBackend default is 4096 and is honoured when given).
    parallelism / pool: accepted for signature compatibility with
      LocalBackend (client.py:29-35); the device engine pipelines on streams.
    outputs: "host" (StreamFile, default) or "device" (DeviceStream).
    """

    parallelism: int = 1
    chunk_size: int | None = None
    pool: str = "thread"
    device: object = None
    stream: object = None
    outputs: str = "host"


LocalBackend = CudaBackend


def _checked_inputs(program, inputs: dict) -> dict:
    free_in = {fp.stream: fp for fp in free_points(program) if fp.direction is Direction.INPUT}
    missing = free_in.keys() - inputs.keys()
    if missing:
        raise ClientError(f"missing input stream {sorted(missing)[0]!r} (free input point)")
    extra = inputs.keys() - free_in.keys()
    if extra:
        raise ClientError(f"{sorted(extra)[0]!r} is not a free input point")
    return free_in


def run(backend: CudaBackend | None, program, inputs: dict) -> dict:
    """Execute ``program`` over whole input streams; blocking for host outputs."""
    import torch

    from ._torch import require_cuda, to_device
    from .executor import chunk_arrays, plan, run_stream

    backend = backend or CudaBackend()
    if not isinstance(backend, CudaBackend):
        raise ClientError(f"unsupported backend {type(backend).__name__}; use CudaBackend")
    program = as_program(program)
    free_in = _checked_inputs(program, inputs)
    p = plan(program, backend.chunk_size, device=backend.device)
    dev = p.device
    require_cuda(dev)
    arrays, counts = {}, set()
    for name, fp in free_in.items():
        sf = inputs[name]
        if sf.data != fp.data:
            raise ClientError(f"stream {name!r} carries {sf.data}, the free point wants {fp.data}")
        if name not in p.broadcast:
            counts.add(sf.count)
        if isinstance(sf, DeviceStream):
            arrays[name] = sf.tensor if sf.tensor.device == dev else sf.tensor.to(dev)
        elif isinstance(sf, StreamFile):
            arrays[name] = to_device(sf.values, dev)
        else:
            raise ClientError(f"stream {name!r}: expected StreamFile or DeviceStream")
    if len(counts) > 1:
        raise ClientError(f"input streams disagree on element count: {sorted(counts)}")
    parts: dict[str, list] = {fp.stream: [] for fp in p.free_outputs}

    def collect(chunk):
        for name, buf in chunk.buffers.items():
            parts[name].append(buf)

    stream = backend.stream
    with torch.cuda.device(dev):
        run_stream(p, chunk_arrays(p, arrays), writer=collect, workers=backend.parallelism,
                   pool=backend.pool, stream=stream)
        out = {}
        for fp in p.free_outputs:
            bufs = parts[fp.stream]
            from ._torch import torch_dtype
            t = (bufs[0] if len(bufs) == 1 else torch.cat(bufs)) if bufs else \
                torch.zeros(0, dtype=torch_dtype(fp.data), device=dev)
            out[fp.stream] = DeviceStream(fp.data, t) if backend.outputs == "device" else \
                StreamFile(fp.data, t.cpu().numpy())
    return out
