"""paper_1203_4938_b200 — B200-native FFT and block-compression nodes for the
arXiv 1203.4938 data-flow platform.

The graph/node/edge API mirrors the reference package ``dpp``
(/root/reference/pkg/src/dpp/__init__.py:12-35): the same Program document
format and ids, stream names and ``run(backend, program, inputs)`` contract.
Nodes execute as hand-written sm_100a kernels behind the C ABI in
``include/dpp_b200.h`` (``libdpp_b200.so``); PyTorch only provides device
buffers and streams.  Importing the graph API needs neither torch nor a GPU;
executing a program needs both, and fails loudly without them.
"""

__version__ = "0.1.0"

from .types import DataType, Direction, IOPoint, parse_type_name
from .model import (Arrow, FreePoint, Instance, Node, Program, ValidationReport, Violation,
                    as_program, free_points, parse_program, program_id, serialize_program,
                    topological_order, validate)
from .wire import DeviceStream, StreamFile
from .client import CudaBackend, LocalBackend, run
from .errors import (ClientError, DeviceError, DppError, EngineRuntimeError, KernelRuntimeError,
                     NativeLibraryError, PlanError, ProgramFormatError)


def __getattr__(name):  # executor symbols need torch: import lazily
    if name in ("ExecutionPlan", "Chunk", "RunResult", "plan", "run_chunk", "run_stream",
                "chunk_arrays", "DEFAULT_CHUNK_SIZE"):
        from . import executor
        return getattr(executor, name)
    raise AttributeError(name)


__all__ = [
    "DataType", "Direction", "IOPoint", "parse_type_name",
    "Node", "Instance", "Arrow", "Program", "FreePoint", "Violation", "ValidationReport",
    "parse_program", "serialize_program", "validate", "topological_order", "program_id",
    "free_points", "as_program",
    "ExecutionPlan", "Chunk", "RunResult", "plan", "run_chunk", "run_stream", "chunk_arrays",
    "DEFAULT_CHUNK_SIZE", "StreamFile", "DeviceStream", "CudaBackend", "LocalBackend", "run",
    "DppError", "ProgramFormatError", "KernelRuntimeError", "PlanError", "EngineRuntimeError",
    "ClientError", "DeviceError", "NativeLibraryError", "__version__",
]
