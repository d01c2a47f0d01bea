"""Golden outputs of the REFERENCE kernel evaluator for the JIT corpus.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_jit_golden.py

For every case of tests/jit_corpus.py the reference front end
(dpp.kernel.compile_kernel) and evaluator (dpp.kernel.run_lanes, one lockstep
batch: gids 0..items-1, global size = items) run on seeded inputs; outputs
(zero-filled first, as the engine hands them) or the raised fault (message,
work-item) go to jit_golden.npz / jit_golden.json.  Ill-typed cases record the
reference's type-check message.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))


def main() -> None:
    from dpp.errors import KernelError, KernelRuntimeError
    from dpp.kernel import compile_kernel, run_lanes
    from dpp.types import DataType, Direction, IOPoint

    from jit_corpus import CASES, make_inputs

    arrays, meta = {}, {}
    for case in CASES:
        name = case["name"]
        io = {p: IOPoint(p, DataType(b, w), Direction.INPUT if d == "in" else Direction.OUTPUT)
              for p, (b, w, d) in case["io"].items()}
        try:
            k = compile_kernel(case["body"], io)
        except KernelError as exc:
            meta[name] = {"compile_error": str(exc)}
            continue
        items = case["items"]
        ins = make_inputs(case)
        outs = {p: np.zeros(items * w, DataType(b, w).dtype) for p, (b, w, d) in case["io"].items() if d == "out"}
        for p, v in ins.items():
            arrays[f"{name}/in/{p}"] = v
        try:
            run_lanes(k, np.arange(items, dtype=np.int32), items, dict(ins), outs)
            meta[name] = {"ok": True}
            for p, v in outs.items():
                arrays[f"{name}/out/{p}"] = v
        except KernelRuntimeError as exc:
            meta[name] = {"fault": str(exc).split(" (work-item")[0], "work_item": exc.work_item}
    # the reference's own application nodes (apps/fft.py:86-117, apps/imgc.py:128-185)
    from dpp.apps import fft as rfft
    from dpp.apps import imgc as rimgc
    apps = [("leaf1", rfft.leaf_kernel(1), 999), ("leaf2", rfft.leaf_kernel(2), 999),
            ("leaf3", rfft.leaf_kernel(3), 999)]
    for pname, prog, items in (("ycbcr", rimgc.ycbcr_program(), 1024), ("boxdown", rimgc.chroma_down_program(), 700),
                               ("gradient", rimgc.gradient_program(32, 16), 512),
                               ("vq", rimgc.vq_program(16), 300)):
        (node,) = prog.kernels.values()
        apps.append((pname, node, items))
    rng = np.random.default_rng(1203)
    for pname, node, items in apps:
        name = "app_" + pname
        io = {pt.name: pt for pt in node.io}
        k = compile_kernel(node.body, io)
        ins = {}
        for pt in node.io:
            if pt.is_input:
                n = items * pt.data.width
                ins[pt.name] = (rng.integers(0, 256, n).astype(pt.data.dtype) if pt.data.is_integer
                                else (rng.standard_normal(n) * 10).astype(np.float32))
        outs = {pt.name: np.zeros(items * pt.data.width, pt.data.dtype) for pt in node.io if not pt.is_input}
        run_lanes(k, np.arange(items, dtype=np.int32), items, dict(ins), outs)
        meta[name] = {"ok": True, "app": True, "items": items, "body": node.body,
                      "io": {pt.name: [pt.data.base, pt.data.width, "in" if pt.is_input else "out"]
                             for pt in node.io}}
        for p_, v in ins.items():
            arrays[f"{name}/in/{p_}"] = v
        for p_, v in outs.items():
            arrays[f"{name}/out/{p_}"] = v
    np.savez_compressed(HERE / "jit_golden.npz", **arrays)
    (HERE / "jit_golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print(len(CASES), "cases;", sum("ok" in m for m in meta.values()), "ok,",
          sum("fault" in m for m in meta.values()), "faults,", sum("compile_error" in m for m in meta.values()),
          "compile errors")


if __name__ == "__main__":
    main()
