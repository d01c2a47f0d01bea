"""The node-body language, compiled to sm_100a instead of interpreted.

Same front end contract as the reference's dpp.kernel
(/root/reference/pkg/src/dpp/kernel: lexer.py, parser.py, typecheck.py) —
tokens with 1-based positions, the SPEC grammar with C precedence, the
OpenCL-1.0-style typing rules — written from SPEC.md (module kernel-lang).
Instead of the lockstep numpy evaluator (interp.py) the typed body is
translated to CUDA C (``codegen``) and compiled at plan time with NVRTC for
sm_100a (``jit``), one thread per work-item, with the interpreter's
arithmetic (binary32 without contraction, two's-complement wrap), bounds
faults, integer-division faults and instruction budget.
"""

from .lexer import Token, scan, tokenize
from .parser import parse_body
from .typecheck import TypedKernel, compile_kernel, typecheck

__all__ = ["Token", "scan", "tokenize", "parse_body", "TypedKernel", "typecheck", "compile_kernel"]
