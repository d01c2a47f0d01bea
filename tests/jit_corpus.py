"""Kernel-language corpus for the JIT and its input recipe.

Each case: body, io {point: (base, width, "in"|"out")}, work-item count,
optional integer input range and float scale, and whether the result must be
bit-exact (transcendental builtins are compared within a few ulp).  Golden
outputs come from the reference evaluator (tests/golden/make_jit_golden.py).
"""

from __future__ import annotations

import zlib

import numpy as np

_I = "int i = get_global_id(0);\n"

CASES = [
    {"name": "adder", "body": _I + "z[i] = x[i] + y[i];",
     "io": {"x": ("float", 1, "in"), "y": ("float", 1, "in"), "z": ("float", 1, "out")}, "items": 1000},
    {"name": "fan", "body": _I + "x[i] = z[i].x;\ny[i] = z[i].y;",
     "io": {"z": ("float", 2, "in"), "x": ("float", 1, "out"), "y": ("float", 1, "out")}, "items": 777},
    {"name": "rot_int", "body": _I + "y[i] = x[i] << 16;",
     "io": {"x": ("int", 1, "in"), "y": ("int", 1, "out")}, "items": 500},
    {"name": "rot_float_ill_typed", "body": _I + "y[i] = x[i] << 16;",
     "io": {"x": ("float", 1, "in"), "y": ("float", 1, "out")}, "items": 4},
    {"name": "int_ops", "items": 2000, "lo": -1000000, "hi": 1000000,
     "body": _I + "int a = x[i]; int b = y[i];\n"
             "int d = b == 0 ? 7 : b;\n"
             "z[i] = (int4)(a / d, a % d, (a * b) ^ (a >> 3), ~a | (b & 0xff));",
     "io": {"x": ("int", 1, "in"), "y": ("int", 1, "in"), "z": ("int", 4, "out")}},
    {"name": "int_wrap", "items": 1000, "lo": -2147483648, "hi": 2147483647,
     "body": _I + "int a = x[i];\nz[i] = (int2)(a * 65599 + 12345, -a - 1);",
     "io": {"x": ("int", 1, "in"), "z": ("int", 2, "out")}},
    {"name": "int_min_div", "items": 8, "lo": -2147483648, "hi": -2147483640,
     "body": _I + "int a = x[i];\nz[i] = (int2)(a / -1, a % -1);",
     "io": {"x": ("int", 1, "in"), "z": ("int", 2, "out")}},
    {"name": "uint_ops", "items": 1500, "lo": 0, "hi": 4294967295,
     "body": _I + "uint a = x[i];\nuint b = y[i] | (uint)(1);\n"
             "z[i] = (uint4)(a / b, a % b, a - b * (uint)(3), (a >> 5) + (b << 7));",
     "io": {"x": ("uint", 1, "in"), "y": ("uint", 1, "in"), "z": ("uint", 4, "out")}},
    {"name": "small_ints", "items": 1024, "lo": -128, "hi": 127,
     "body": _I + "char a = x[i];\nuchar u = (uchar)(a);\nshort s = (short)(a) * (short)(300);\n"
             "ushort us = (ushort)(s);\n"
             "z[i] = (int4)((int)(a + a + a), (int)(u + u), (int)(s), (int)(us >> 3));",
     "io": {"x": ("char", 1, "in"), "z": ("int", 4, "out")}},
    {"name": "long_ops", "items": 1000, "lo": -9000000000000000000, "hi": 9000000000000000000,
     "body": _I + "long a = x[i];\nlong b = y[i] == 0 ? 3 : y[i];\n"
             "w[i] = (long2)(a * 6364136223846793005 + 1442695040888963407, a / b);\n"
             "u[i] = (ulong)(a) >> 33;",
     "io": {"x": ("long", 1, "in"), "y": ("long", 1, "in"), "w": ("long", 2, "out"), "u": ("ulong", 1, "out")}},
    {"name": "shifts_masked", "items": 300, "lo": -64, "hi": 64,
     "body": _I + "int s = y[i];\nz[i] = (int2)(x[i] << s, x[i] >> s);",
     "io": {"x": ("int", 1, "in"), "y": ("int", 1, "in"), "z": ("int", 2, "out")}},
    {"name": "promote_mixed", "items": 900, "lo": -300, "hi": 300,
     "body": _I + "int a = x[i];\nfloat f = y[i];\nuchar c = (uchar)(a);\n"
             "z[i] = (float4)(a + f, f / a, (float)(c + 1), f * 3);",
     "io": {"x": ("int", 1, "in"), "y": ("float", 1, "in"), "z": ("float", 4, "out")}},
    {"name": "float_to_int_casts", "items": 800, "scale": 1000.0,
     "body": _I + "float f = x[i];\nz[i] = (int4)((int)(f), (int)(-f), (int)((uchar)((int)(f))), (int)(floor(f)));",
     "io": {"x": ("float", 1, "in"), "z": ("int", 4, "out")}},
    {"name": "compare_logic", "items": 1000, "scale": 2.0,
     "body": _I + "float a = x[i];\nfloat b = y[i];\n"
             "int c = (a < b) + 2 * (a >= 0.5f && b < 0.0f) + 4 * (a == b || !(a != a)) + 8 * (a > b ? 1 : 0);\n"
             "z[i] = c;",
     "io": {"x": ("float", 1, "in"), "y": ("float", 1, "in"), "z": ("int", 1, "out")}},
    {"name": "guarded_reads", "items": 513,
     "body": _I + "int n = get_global_size(0);\n"
             "float nxt = i + 1 < n ? x[i + 1] : 0.0f;\n"
             "float prv = (i > 0 && x[i - 1] > 0.0f) ? x[i - 1] : -1.0f;\n"
             "z[i] = nxt - prv;",
     "io": {"x": ("float", 1, "in"), "z": ("float", 1, "out")}},
    {"name": "for_sum_sequential", "items": 400, "scale": 100.0,
     "body": _I + "float s = 0.0f;\nfor (int k = 0; k < 16; k = k + 1) {\n"
             "  if (k == 0) { s = blk[i].s0; } else { s = s + (k < 8 ? (float)(k) * 0.1f : blk[i].sF); }\n}\n"
             "avg[i] = s * 0.0625f;",
     "io": {"blk": ("float", 16, "in"), "avg": ("float", 1, "out")}},
    {"name": "vectors", "items": 600,
     "body": _I + "float4 a = x[i];\nfloat4 b = a * 2.0f - (float4)(1.0f, 2.0f, 3.0f, 4.0f);\n"
             "b.y = -b.w;\nfloat4 c = b / a;\n"
             "z[i] = c;\nz[i].x = a.x * b.z + a.y;",
     "io": {"x": ("float", 4, "in"), "z": ("float", 4, "out")}},
    {"name": "dots", "items": 700, "scale": 30.0,
     "body": _I + "z[i] = (float4)(dot(a[i], b[i]), dot(c[i], c[i]), dot(e[i], e[i]), dot(f[i], f[i]));",
     "io": {"a": ("float", 2, "in"), "b": ("float", 2, "in"), "c": ("float", 4, "in"),
            "e": ("float", 8, "in"), "f": ("float", 16, "in"), "z": ("float", 4, "out")}},
    {"name": "exact_builtins", "items": 900, "scale": 50.0,
     "body": _I + "float a = x[i];\nfloat b = y[i];\n"
             "z[i] = (float8)(fabs(a), floor(a), sqrt(fabs(a)), fmin(a, b), fmax(a, b), "
             "(float)(min((int)(a), (int)(b))), (float)(max((int)(a), (int)(b))), (float)(abs((int)(a))));",
     "io": {"x": ("float", 1, "in"), "y": ("float", 1, "in"), "z": ("float", 8, "out")}},
    {"name": "transcendental", "items": 1000, "scale": 3.0, "exact": False,
     "body": _I + "float a = x[i];\nz[i] = (float8)(sin(a), cos(a), exp(a), log(fabs(a) + 1.0f), "
             "pow(fabs(a), 1.5f), sin(a * M_PI_F), sqrt(exp(a)), cos(a) * sin(a));",
     "io": {"x": ("float", 1, "in"), "z": ("float", 8, "out")}},
    {"name": "partial_writes", "items": 1001,
     "body": _I + "if (i % 2 == 0) { y[i] = x[i] + 1.0f; }\nif (i % 5 == 0) { y[i] = 5.0f; }",
     "io": {"x": ("float", 1, "in"), "y": ("float", 1, "out")}},
    {"name": "nested_loops_budget_ok", "items": 64,
     "body": _I + "int acc = 0;\nfor (int a = 0; a < 10; a = a + 1) { for (int b = 0; b < a; b = b + 1) "
             "{ acc = acc + a * b + x[i]; } }\ny[i] = acc;",
     "io": {"x": ("int", 1, "in"), "y": ("int", 1, "out")}, "lo": -5, "hi": 5},
    {"name": "scatter_reverse", "items": 333,
     "body": _I + "int n = get_global_size(0);\ny[n - 1 - i] = x[i] * 2.0f;",
     "io": {"x": ("float", 1, "in"), "y": ("float", 1, "out")}},
    {"name": "fault_read_oob", "items": 300,
     "body": _I + "y[i] = x[i] + x[i + 1];",
     "io": {"x": ("float", 1, "in"), "y": ("float", 1, "out")}},
    {"name": "fault_write_oob", "items": 200,
     "body": _I + "y[i] = x[i];\nif (i > 150) { y[i * 2] = 1.0f; }",
     "io": {"x": ("float", 1, "in"), "y": ("float", 1, "out")}},
    {"name": "fault_div_zero", "items": 100, "lo": 0, "hi": 3,
     "body": _I + "y[i] = 10 / x[i];",
     "io": {"x": ("int", 1, "in"), "y": ("int", 1, "out")}},
    {"name": "fault_mod_zero_late", "items": 50, "lo": 1, "hi": 9,
     "body": _I + "int a = x[i];\nfor (int k = 0; k < 3; k = k + 1) { a = a - 1; }\ny[i] = 100 % (a + 2);",
     "io": {"x": ("int", 1, "in"), "y": ("int", 1, "out")}},
    # divergent faults: the reported work-item is the lockstep evaluator's
    # (then-branch before else-branch, loop iteration k for every live lane
    # before k+1), not the one with the fewest statements executed
    {"name": "fault_divergent_branches", "items": 50,
     "body": _I + "if (i < 2) { float a = 1.0f; y[i + 1000] = a; } else { y[i + 1000] = 0.0f; }",
     "io": {"x": ("float", 1, "in"), "y": ("float", 1, "out")}},
    {"name": "fault_divergent_path_length", "items": 64,
     "body": _I + "float a = 0.0f;\nif (i % 2 == 0) { a = 1.0f; a = a + 1.0f; a = a * 2.0f; }\n"
             "y[i + (i >= 10 ? 1000 : 0)] = a;",
     "io": {"x": ("float", 1, "in"), "y": ("float", 1, "out")}},
    {"name": "fault_divergent_loop", "items": 16,
     "body": _I + "int n = (i == 7) ? 6 : 1;\nfor (int k = 0; k < n; k = k + 1) { if (k == 5) { y[i + 1000] = 1.0f; } }\n"
             "y[i + (i == 3 ? 1000 : 0)] = 2.0f;",
     "io": {"x": ("float", 1, "in"), "y": ("float", 1, "out")}},
    {"name": "fault_in_loop_condition", "items": 40, "lo": 0, "hi": 3,
     "body": _I + "int acc = 0;\nfor (int k = 0; k < x[i + k * (i % 3)]; k = k + 1) { acc = acc + k; }\ny[i] = acc;",
     "io": {"x": ("int", 1, "in"), "y": ("int", 1, "out")}},
    {"name": "type_error_write_input", "items": 4, "body": _I + "x[i] = 1.0f;",
     "io": {"x": ("float", 1, "in"), "y": ("float", 1, "out")}},
    {"name": "type_error_narrowing", "items": 4, "body": _I + "int a = x[i];\ny[i] = a;",
     "io": {"x": ("float", 1, "in"), "y": ("int", 1, "out")}},
    {"name": "syntax_error", "items": 4, "body": _I + "y[i] = (x[i] + ;",
     "io": {"x": ("float", 1, "in"), "y": ("float", 1, "out")}},
    {"name": "uchar4_pixels", "items": 640, "lo": 0, "hi": 255,
     "body": _I + "uchar4 p = rgb[i];\n"
             "yl[i] = 0.299f * (float)(p.x) + 0.587f * (float)(p.y) + 0.114f * (float)(p.z);",
     "io": {"rgb": ("uchar", 4, "in"), "yl": ("float", 1, "out")}},
]


def make_inputs(case) -> dict:
    """Seeded inputs for every input point of ``case`` (flat scalar buffers)."""
    rng = np.random.default_rng(zlib.crc32(case["name"].encode()))
    out = {}
    for p, (base, width, d) in case["io"].items():
        if d != "in":
            continue
        n = case["items"] * width
        if base == "float":
            out[p] = (rng.standard_normal(n) * case.get("scale", 1.0)).astype(np.float32)
        else:
            info = np.iinfo({"char": np.int8, "uchar": np.uint8, "short": np.int16, "ushort": np.uint16,
                             "int": np.int32, "uint": np.uint32, "long": np.int64, "ulong": np.uint64}[base])
            lo = max(case.get("lo", info.min), info.min)
            hi = min(case.get("hi", info.max), info.max)
            out[p] = rng.integers(lo, hi, size=n, endpoint=True, dtype=np.int64 if base != "ulong" else np.uint64) \
                .astype(info.dtype) if base not in ("long", "ulong") else \
                rng.integers(lo, hi, size=n, endpoint=True, dtype=info.dtype)
    return out
