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
    np.savez_compressed(HERE / "jit_golden.npz", **arrays)
    (HERE / "jit_golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print(len(CASES), "cases;", sum("ok" in m for m in meta.values()), "ok,",
          sum("fault" in m for m in meta.values()), "faults,", sum("compile_error" in m for m in meta.values()),
          "compile errors")


if __name__ == "__main__":
    main()
