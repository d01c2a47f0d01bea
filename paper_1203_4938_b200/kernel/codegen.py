"""Typed kernel body -> CUDA C for one thread per work-item.

Semantics follow the reference evaluator (/root/reference/pkg/src/dpp/kernel/
interp.py), restated per operation:

* every operand is converted to the operator's annotated type first
  (``_cast`` = numpy ``astype``); scalars broadcast against vectors;
* binary32 arithmetic is IEEE round-to-nearest with no contraction
  (``__fadd_rn`` ... ``__fdiv_rn``; NVRTC also runs with ``-fmad=false``);
* integer + - * and unary minus wrap (two's complement, done in the unsigned
  type); / and % truncate toward zero (the evaluator's floor-divide fix-up)
  and fault on a zero divisor; MIN / -1 wraps like numpy;
* shift counts are masked to the operand width (``& (bits - 1)``);
* comparisons are done in the promoted ``wide`` type and yield int 0/1;
  ``&&`` / ``||`` / ``?:`` evaluate their right / branch operands only where
  needed (so a guarded out-of-range read does not fault);
* ``dot`` sums the binary32 products in numpy's order: left to right for
  widths 2-4, the pairwise-8 tree (r_j = p_j + p_{j+8}) for 8 and 16;
* ``fmin``/``fmax``/``min``/``max`` are numpy minimum/maximum
  (``a < b || isnan(a) ? a : b``); transcendental builtins use CUDA's
  accurate ``sinf`` ... ``powf`` (within a few ulp of numpy's float32);
* buffer reads and writes are bounds-checked.  Every fault site has a
  position in the lockstep evaluator's order — (loop region, iteration, ...,
  site) of pre-order ids — and the reported fault is the minimum position
  over all work-items, then the lowest work-item, exactly the one the
  reference's lockstep interpreter raises first: the then-branch before the
  else-branch, iteration k of a loop for every live lane before k+1
  (interp.py:118-180).  A normal launch only flags a fault; jit.py then finds
  the minimum one tuple component per re-run and recovers the detail from the
  one faulting work-item;
* every statement a work-item executes counts against the instruction budget
  (per work-item path; the reference counts the frame's lockstep statements,
  which is larger only when lanes diverge inside long loops).
"""

from __future__ import annotations

import numpy as np

from ..types import DataType
from . import ast
from .typecheck import TypedKernel

__all__ = ["generate", "CTYPES", "FAULT_INDEX", "FAULT_DIV", "FAULT_MOD", "FAULT_BUDGET"]

CTYPES = {"char": "signed char", "uchar": "unsigned char", "short": "short", "ushort": "unsigned short",
          "int": "int", "uint": "unsigned int", "long": "long long", "ulong": "unsigned long long",
          "float": "float"}
_UTYPES = {1: "unsigned char", 2: "unsigned short", 4: "unsigned int", 8: "unsigned long long"}
FAULT_INDEX, FAULT_DIV, FAULT_MOD, FAULT_BUDGET = 1, 2, 3, 4

_PRELUDE = r"""
// A fault site's position in the lockstep evaluator's order (interp.py:118-
// 180: statements run for every active lane before the next one starts, the
// then-branch before the else-branch, loop iteration k for all live lanes
// before iteration k+1): the tuple (loop region, iteration, ..., site) of
// pre-order ids, compared lexicographically, then the work-item.  A normal
// launch only flags a fault; diagnosis passes (jit.py) re-run the node and
// find the minimum tuple one component per pass, then the lowest work-item.
#define DPP_FAULT(code, pt, val, ...) do { \
    const long long tup_[] = {__VA_ARGS__}; \
    dpp_fault(fault, diag, mode, prefix, gid, code, pt, (long long)(val), tup_, \
              (int)(sizeof(tup_) / sizeof(long long))); return; } while (0)
__device__ __forceinline__ void dpp_fault(unsigned long long* fault, long long* diag, int mode,
                                          const long long* prefix, long long gid, int code, int pt, long long val,
                                          const long long* tup, int len) {
  if (mode < 0) {  // normal launch: only "a fault happened"
    atomicMin(fault, 0ULL);
    if (diag) { diag[0] = code; diag[1] = pt; diag[2] = val; }
    return;
  }
  for (int j = 0; j < mode; ++j)
    if (j >= len || tup[j] != prefix[j]) return;  // not on the minimum's path
  atomicMin(fault, (unsigned long long)(mode < len ? tup[mode] : gid));
}
__device__ __forceinline__ float dpp_fmin(float a, float b) { return (a < b || isnan(a)) ? a : b; }
__device__ __forceinline__ float dpp_fmax(float a, float b) { return (a > b || isnan(a)) ? a : b; }
"""


def _f32_bits(x: float) -> str:
    return f"__int_as_float(0x{int(np.float32(x).view(np.uint32)):08x})"


class _Gen:
    def __init__(self, k: TypedKernel, budget: int):
        self.k = k
        self.budget = budget
        self.lines: list[str] = []
        self.ind = 1
        self.n = 0
        self.points = list(k.io.values())
        self.pid = {p.name: i for i, p in enumerate(self.points)}
        self.scopes: list[dict] = [{}]
        self.pre = 0                   # pre-order ids of statements, fault sites and loop regions
        self.loops: list[tuple] = []   # enclosing loops: (region id, iteration counter)
        self.sites: set[int] = set()   # ids that end a fault tuple

    def site(self) -> str:
        """A new fault site: its lockstep tuple as DPP_FAULT's trailing arguments."""
        self.pre += 1
        self.sites.add(self.pre)
        parts = []
        for region, it in self.loops:
            parts += [str(region), it]
        return ", ".join(parts + [str(self.pre)])

    # -- emission helpers -------------------------------------------------
    def emit(self, line: str) -> None:
        self.lines.append("  " * self.ind + line)

    def tmp(self, ctype: str, value: str) -> str:
        self.n += 1
        name = f"t{self.n}"
        self.emit(f"{ctype} {name} = {value};")
        return name

    def open(self, head: str = "{") -> None:
        self.emit(head)
        self.ind += 1

    def close(self, tail: str = "}") -> None:
        self.ind -= 1
        self.emit(tail)

    def var(self, name: str) -> tuple:
        for sc in reversed(self.scopes):
            if name in sc:
                return sc[name]
        raise KeyError(name)  # pragma: no cover (typecheck guarantees)

    # -- conversions ---------------------------------------------------------
    @staticmethod
    def conv(v: str, src: DataType, dst: DataType) -> str:
        s, d = src.base, dst.base
        if s == d:
            return v
        ct = CTYPES[d]
        if dst.is_float:
            if src.scalar_size <= 2:
                return f"(float)({v})"
            fn = {"int": "__int2float_rn", "uint": "__uint2float_rn", "long": "__ll2float_rn",
                  "ulong": "__ull2float_rn"}[s]
            return f"{fn}({v})"
        return f"(({ct})({v}))"

    def cast(self, vals: list, src: DataType, dst: DataType) -> list:
        """Convert to dst's base and broadcast a scalar to dst's width."""
        out = [self.conv(v, src, dst) for v in vals]
        if len(out) == 1 and dst.width > 1:
            t = self.tmp(CTYPES[dst.base], out[0])
            return [t] * dst.width
        return out

    # -- expressions --------------------------------------------------------
    def expr(self, e) -> list:
        m = getattr(self, "e_" + type(e).__name__)
        return m(e)

    def e_IntLit(self, e):
        t = e.type
        suffix = "ll" if t.base in ("long", "ulong") else ""
        return [f"(({CTYPES[t.base]}){e.value}{suffix})"]

    def e_FloatLit(self, e):
        return [_f32_bits(e.value)]

    def e_Ident(self, e):
        if e.name == "M_PI_F":
            return [_f32_bits(np.pi)]
        names, _ = self.var(e.name)
        return list(names)

    def gather(self, name: str, index, comp):
        p = self.k.io[name]
        i = self.index_value(index, name)
        w = p.data.width
        ptr = f"b{self.pid[name]}"
        if comp is not None:
            return [self.tmp(CTYPES[p.data.base], f"{ptr}[{i} * {w} + {comp}]")]
        if w == 1:
            return [self.tmp(CTYPES[p.data.base], f"{ptr}[{i}]")]
        return [self.tmp(CTYPES[p.data.base], f"{ptr}[{i} * {w} + {c}]") for c in range(w)]

    def index_value(self, index, name: str) -> str:
        (iv,) = self.expr(index)
        i = self.tmp("long long", f"(long long)({iv})")
        self.emit(f"if ({i} < 0 || {i} >= n{self.pid[name]}) "
                  f"DPP_FAULT({FAULT_INDEX}, {self.pid[name]}, {i}, {self.site()});")
        return i

    def e_Index(self, e):
        return self.gather(e.name, e.index, None)

    def e_Comp(self, e):
        if isinstance(e.base, ast.Index):
            return self.gather(e.base.name, e.base.index, e.comp)
        return [self.expr(e.base)[e.comp]]

    def e_Unary(self, e):
        src = e.operand.type
        vals = self.expr(e.operand)
        if e.op == "!":
            return [self.tmp("int", f"(({vals[0]}) == 0)")]
        t = e.type
        ct = CTYPES[t.base]
        vals = self.cast(vals, src, t)
        if e.op == "~":
            return [self.tmp(ct, f"({ct})(~({v}))") for v in vals]
        if t.is_float:
            return [self.tmp(ct, f"-({v})") for v in vals]
        ut = _UTYPES[t.scalar_size]
        return [self.tmp(ct, f"({ct})(({ut})0 - ({ut})({v}))") for v in vals]

    def e_Binary(self, e):
        op = e.op
        if op in ("&&", "||"):
            (a,) = self.expr(e.left)
            r = self.tmp("int", "0")
            self.open(f"if (({a}) {'!=' if op == '&&' else '=='} 0) {{")
            (b,) = self.expr(e.right)
            self.emit(f"{r} = (({b}) != 0);")
            self.close("}" if op == "&&" else "} else {")
            if op == "||":
                self.ind += 1
                self.emit(f"{r} = 1;")
                self.close()
            return [r]
        if op in ("==", "!=", "<", "<=", ">", ">="):
            w = e.wide
            (a,) = self.cast(self.expr(e.left), e.left.type, w)
            (b,) = self.cast(self.expr(e.right), e.right.type, w)
            return [self.tmp("int", f"(({a}) {op} ({b}))")]
        t = e.type
        ct = CTYPES[t.base]
        la = self.expr(e.left)
        ra = self.expr(e.right)
        if op in ("<<", ">>"):
            bits = t.scalar_size * 8
            la = self.cast(la, e.left.type, t)
            rs = [self.tmp(ct, f"({ct})((long long)({v}) & {bits - 1})") for v in ra]
            if len(rs) == 1 and t.width > 1:
                rs = rs * t.width
            ut = _UTYPES[t.scalar_size]
            if op == "<<":
                return [self.tmp(ct, f"({ct})(({ut})({a}) << ({b}))") for a, b in zip(la, rs)]
            return [self.tmp(ct, f"({ct})(({a}) >> ({b}))") for a, b in zip(la, rs)]
        la = self.cast(la, e.left.type, t)
        ra = self.cast(ra, e.right.type, t)
        out = []
        for a, b in zip(la, ra):
            if t.is_float:
                fn = {"+": "__fadd_rn", "-": "__fsub_rn", "*": "__fmul_rn", "/": "__fdiv_rn"}[op]
                out.append(self.tmp("float", f"{fn}({a}, {b})"))
            elif op in ("+", "-", "*"):
                ut = _UTYPES[t.scalar_size]
                out.append(self.tmp(ct, f"({ct})(({ut})({a}) {op} ({ut})({b}))"))
            elif op in ("/", "%"):
                code = FAULT_DIV if op == "/" else FAULT_MOD
                self.emit(f"if (({b}) == 0) DPP_FAULT({code}, -1, 0, {self.site()});")
                if t.is_signed and t.scalar_size >= 4:
                    ut = _UTYPES[t.scalar_size]
                    alt = f"({ct})(({ut})0 - ({ut})({a}))" if op == "/" else f"({ct})0"
                    out.append(self.tmp(ct, f"(({b}) == ({ct})-1) ? {alt} : ({ct})(({a}) {op} ({b}))"))
                else:
                    out.append(self.tmp(ct, f"({ct})(({a}) {op} ({b}))"))
            else:  # & | ^
                out.append(self.tmp(ct, f"({ct})(({a}) {op} ({b}))"))
        return out

    def e_Ternary(self, e):
        t = e.type
        ct = CTYPES[t.base]
        (c,) = self.expr(e.cond)
        rs = [self.tmp(ct, f"({ct})0") for _ in range(t.width)]
        self.open(f"if (({c}) != 0) {{")
        for r, v in zip(rs, self.cast(self.expr(e.then), e.then.type, t)):
            self.emit(f"{r} = {v};")
        self.close("} else {")
        self.ind += 1
        for r, v in zip(rs, self.cast(self.expr(e.other), e.other.type, t)):
            self.emit(f"{r} = {v};")
        self.close()
        return rs

    def e_Call(self, e):
        name = e.name
        if name == "get_global_id":
            return ["((int)gid)"]
        if name == "get_global_size":
            return ["((int)gsize)"]
        t = e.type
        if name == "dot":
            a = self.expr(e.args[0])
            b = self.expr(e.args[1])
            p = [self.tmp("float", f"__fmul_rn({x}, {y})") for x, y in zip(a, b)]
            w = len(p)
            if w <= 4:
                acc = p[0]
                for q in p[1:]:
                    acc = self.tmp("float", f"__fadd_rn({acc}, {q})")
                return [acc]
            r = [p[j] if w == 8 else self.tmp("float", f"__fadd_rn({p[j]}, {p[j + 8]})") for j in range(8)]
            s01 = self.tmp("float", f"__fadd_rn({r[0]}, {r[1]})")
            s23 = self.tmp("float", f"__fadd_rn({r[2]}, {r[3]})")
            s45 = self.tmp("float", f"__fadd_rn({r[4]}, {r[5]})")
            s67 = self.tmp("float", f"__fadd_rn({r[6]}, {r[7]})")
            lo = self.tmp("float", f"__fadd_rn({s01}, {s23})")
            hi = self.tmp("float", f"__fadd_rn({s45}, {s67})")
            return [self.tmp("float", f"__fadd_rn({lo}, {hi})")]
        ct = CTYPES[t.base]
        if len(e.args) == 1:
            vals = self.expr(e.args[0])
            if name == "abs":
                ut = _UTYPES[t.scalar_size]
                if t.is_signed:
                    return [self.tmp(ct, f"(({v}) < 0) ? ({ct})(({ut})0 - ({ut})({v})) : ({v})") for v in vals]
                return vals
            fn = {"sin": "sinf", "cos": "cosf", "sqrt": "__fsqrt_rn", "fabs": "fabsf", "floor": "floorf",
                  "exp": "expf", "log": "logf"}[name]
            return [self.tmp("float", f"{fn}({v})") for v in vals]
        a = self.cast(self.expr(e.args[0]), e.args[0].type, t)
        b = self.cast(self.expr(e.args[1]), e.args[1].type, t)
        out = []
        for x, y in zip(a, b):
            if name == "pow":
                out.append(self.tmp("float", f"powf({x}, {y})"))
            elif name == "fmin":
                out.append(self.tmp("float", f"dpp_fmin({x}, {y})"))
            elif name == "fmax":
                out.append(self.tmp("float", f"dpp_fmax({x}, {y})"))
            elif name == "min":
                out.append(self.tmp(ct, f"(({x}) < ({y})) ? ({x}) : ({y})"))
            else:  # max
                out.append(self.tmp(ct, f"(({x}) > ({y})) ? ({x}) : ({y})"))
        return out

    def e_Ctor(self, e):
        t = e.ctype
        out = []
        for a in e.args:
            (v,) = self.expr(a)
            out.append(self.tmp(CTYPES[t.base], self.conv(v, a.type, t.scalar)))
        return out

    # -- statements ---------------------------------------------------------
    def count(self) -> None:
        self.emit(f"if (++ops > {self.budget}LL) DPP_FAULT({FAULT_BUDGET}, -1, 0, {self.site()});")

    def stmt(self, s) -> None:
        self.count()
        getattr(self, "s_" + type(s).__name__)(s)

    def s_Decl(self, s):
        t = s.dtype
        ct = CTYPES[t.base]
        if s.init is not None:
            vals = self.cast(self.expr(s.init), s.init.type, t)
        else:
            vals = [f"({ct})0"] * t.width
        self.n += 1
        names = [f"v{self.n}_{s.name}_{c}" for c in range(t.width)]
        for nm, v in zip(names, vals):
            self.emit(f"{ct} {nm} = {v};")
        self.scopes[-1][s.name] = (names, t)

    def s_Assign(self, s):
        tg = s.target
        if tg.name in self.k.io:
            p = self.k.io[tg.name]
            i = self.index_value(tg.index, tg.name)
            w = p.data.width
            ptr = f"b{self.pid[tg.name]}"
            if tg.comp is not None:
                (v,) = self.cast(self.expr(s.value), s.value.type, p.data.scalar)
                self.emit(f"{ptr}[{i} * {w} + {tg.comp}] = {v};")
            else:
                vals = self.cast(self.expr(s.value), s.value.type, p.data)
                for c, v in enumerate(vals):
                    self.emit(f"{ptr}[{i} * {w} + {c}] = {v};")
            return
        names, t = self.var(tg.name)
        if tg.comp is not None:
            (v,) = self.cast(self.expr(s.value), s.value.type, t.scalar)
            self.emit(f"{names[tg.comp]} = {v};")
        else:
            vals = self.cast(self.expr(s.value), s.value.type, t)
            for nm, v in zip(names, vals):
                self.emit(f"{nm} = {v};")

    def scoped(self, s) -> None:
        self.open()
        self.scopes.append({})
        self.stmt(s)
        self.scopes.pop()
        self.close()

    def s_If(self, s):
        (c,) = self.expr(s.cond)
        self.open(f"if (({c}) != 0) {{")
        self.scopes.append({})
        self.stmt(s.then)
        self.scopes.pop()
        if s.other is not None:
            self.close("} else {")
            self.ind += 1
            self.scopes.append({})
            self.stmt(s.other)
            self.scopes.pop()
        self.close()

    def s_For(self, s):
        self.open()
        self.scopes.append({})
        if s.init is not None:
            self.stmt(s.init)
        # the iterations form one region after the init: condition, body and
        # update of iteration k run (in lockstep) before iteration k+1
        self.pre += 1
        self.n += 1
        it = f"it{self.n}"
        self.emit(f"long long {it} = 0;")
        self.loops.append((self.pre, it))
        self.open("for (;; ++" + it + ") {")
        (c,) = self.expr(s.cond)
        self.emit(f"if (({c}) == 0) break;")
        self.scoped(s.body)
        self.stmt(s.update)
        self.close()
        self.loops.pop()
        self.scopes.pop()
        self.close()

    def s_Block(self, s):
        self.open()
        self.scopes.append({})
        for x in s.stmts:
            self.stmt(x)
        self.scopes.pop()
        self.close()


def generate(k: TypedKernel, name: str = "dpp_jit_kernel", budget: int = 10_000_000) -> tuple[str, list, set]:
    """CUDA C source, the parameter list and the ids that end a fault tuple.

    Parameters (all 64-bit): one pointer per i/o point (in ``k.io`` order),
    one element count per point, then items, global size, first gid, fault
    word pointer, detail pointer (nullable), diagnosis pass (-1 = normal
    launch) and the pointer to the tuple prefix fixed by earlier passes."""
    g = _Gen(k, budget)
    for x in k.body:
        g.stmt(x)
    params = []
    decl = []
    for i, p in enumerate(g.points):
        const = "const " if p.is_input else ""
        decl.append(f"  {const}{CTYPES[p.data.base]}* __restrict__ b{i} = ({const}{CTYPES[p.data.base]}*)P[{i}];")
        params.append(("ptr", p.name))
    np_ = len(g.points)
    for i in range(np_):
        decl.append(f"  const long long n{i} = (long long)P[{np_ + i}];")
        params.append(("count", g.points[i].name))
    base = 2 * np_
    decl += [f"  const long long items = (long long)P[{base}];",
             f"  const long long gsize = (long long)P[{base + 1}];",
             f"  const long long gid = (long long)P[{base + 2}] + (long long)blockIdx.x * blockDim.x + threadIdx.x;",
             f"  unsigned long long* fault = (unsigned long long*)P[{base + 3}];",
             f"  long long* diag = (long long*)P[{base + 4}];",
             f"  const int mode = (int)(long long)P[{base + 5}];",
             f"  const long long* prefix = (const long long*)P[{base + 6}];",
             f"  if (gid >= (long long)P[{base + 2}] + items) return;",
             "  long long ops = 0;"]
    params += [("items",), ("gsize",), ("gid0",), ("fault",), ("diag",), ("mode",), ("prefix",)]
    src = (_PRELUDE + f'\nstruct dpp_params {{ unsigned long long p[{base + 7}]; }};\n'
           f'extern "C" __global__ void __launch_bounds__(256) {name}(const dpp_params prm) {{\n'
           "  const unsigned long long* P = prm.p;\n" + "\n".join(decl) + "\n" + "\n".join(g.lines) + "\n}\n")
    return src, params, g.sites
