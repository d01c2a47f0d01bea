"""Device data plane (dataplane.pump / serve_run): a loopback run speaking the
reference's frame protocol gives the same bytes as run() on the same plan."""

from __future__ import annotations

import json
import socket
import threading

import numpy as np
import pytest

from conftest import complex_signals, table2_doc

pytestmark = pytest.mark.gpu


def _loopback(program, inputs: dict, chunk_size: int, max_in_flight: int = 3, run_id: str = "run-1",
              client_run_id: str | None = None):
    """Server thread: serve_run on the device; client: the reference client's
    handshake + send/collect.  Returns (outputs, work items, server error)."""
    from paper_1203_4938_b200 import dataplane as dp
    from paper_1203_4938_b200.executor import plan
    from paper_1203_4938_b200.model import free_points
    from paper_1203_4938_b200.types import Direction
    p = plan(program, chunk_size)
    a, b = socket.socketpair()
    result = {}

    def server():
        try:
            result["items"] = dp.serve_run(p, b, run_id, max_in_flight)
        except Exception as exc:  # noqa: BLE001
            result["error"] = exc

    t = threading.Thread(target=server, daemon=True)
    t.start()
    free = free_points(program)
    fin = [fp for fp in free if fp.direction is Direction.INPUT]
    fout = [fp for fp in free if fp.direction is Direction.OUTPUT]
    try:
        a.sendall(dp.encode_handshake(client_run_id or run_id))
        ok, message = dp.read_reply(a)
        if not ok:
            t.join(timeout=30)
            return None, message, result.get("error")
        sender = threading.Thread(target=dp.send_inputs, args=(a, fin, {k: v.values for k, v in inputs.items()},
                                                                  chunk_size), daemon=True)
        sender.start()
        out = dp.collect_outputs(a, fout)
        sender.join(timeout=60)
        t.join(timeout=60)
        return out, result.get("items"), result.get("error")
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("slots", [1, 3])
def test_fft_program_over_the_data_plane_matches_run(cuda, slots):
    from paper_1203_4938_b200 import CudaBackend, DataType, StreamFile, run
    from paper_1203_4938_b200.apps.fft import fft_program
    x = complex_signals(11, (42, 256))  # 10 chunks of 4 signals, then a short one of 2
    sf = StreamFile(DataType("float", 2), x.reshape(-1).view(np.float32))
    ref = run(CudaBackend(chunk_size=1024), fft_program(256), {"0.x": sf})["0.y"].values
    out, items, err = _loopback(fft_program(256), {"0.x": sf}, 1024, slots)
    assert err is None
    assert np.array_equal(out["0.y"].values, ref)
    assert items == 42 * 256


def test_table2_jit_graph_over_the_data_plane(cuda):
    from paper_1203_4938_b200 import DataType, StreamFile, parse_program, run
    prog = parse_program(json.dumps(table2_doc()))
    z = np.random.default_rng(3).standard_normal(2 * 1000).astype(np.float32)
    sf = StreamFile(DataType("float", 2), z)
    ref = run(None, prog, {"0.z": sf})["2.z"].values
    out, items, err = _loopback(prog, {"0.z": sf}, 128)
    assert err is None and np.array_equal(out["2.z"].values, ref)


def test_wrong_run_and_faults_reach_the_client(cuda):
    from paper_1203_4938_b200 import ClientError, DataType, StreamFile
    from paper_1203_4938_b200.errors import ProtocolError
    from paper_1203_4938_b200.apps.fft import fft_program
    sf = StreamFile(DataType("float", 2), complex_signals(1, 512).view(np.float32))
    out, message, err = _loopback(fft_program(256), {"0.x": sf}, 512, client_run_id="other")
    assert out is None and message == "unknown run 'other'" and isinstance(err, ProtocolError)
    # a partial signal faults in the node: the server sends ERROR, the client raises
    sf = StreamFile(DataType("float", 2), complex_signals(1, 384).view(np.float32))
    with pytest.raises(ClientError, match="run failed"):
        _loopback(fft_program(256), {"0.x": sf}, 384)


def test_empty_stream_over_the_data_plane(cuda):
    """No DATA frames at all: END frames only, empty outputs, zero work-items
    (the reference's _assemble_chunks accepts END-only runs)."""
    from paper_1203_4938_b200 import CudaBackend, DataType, StreamFile, run
    from paper_1203_4938_b200.apps.fft import fft_program
    sf = StreamFile(DataType("float", 2), np.zeros(0, np.float32))
    out, items, err = _loopback(fft_program(256), {"0.x": sf}, 1024)
    assert err is None and items == 0 and out["0.y"].values.size == 0
    assert run(CudaBackend(), fft_program(256), {"0.x": sf})["0.y"].values.size == 0


def test_two_input_streams_over_the_data_plane(cuda):
    """One DATA frame per free input per chunk (the reference's adder node,
    x and y both free): chunks assemble only when both have arrived."""
    from paper_1203_4938_b200 import DataType, StreamFile, parse_program, run
    doc = table2_doc()
    doc["nodes"] = [[0, {"kernel": "adder"}]]
    doc["arrows"] = []
    prog = parse_program(json.dumps(doc))
    rng = np.random.default_rng(8)
    xs = StreamFile(DataType("float", 1), rng.standard_normal(3000).astype(np.float32))
    ys = StreamFile(DataType("float", 1), rng.standard_normal(3000).astype(np.float32))
    ref = run(None, prog, {"0.x": xs, "0.y": ys})["0.z"].values
    assert np.array_equal(ref, xs.values + ys.values)
    out, items, err = _loopback(prog, {"0.x": xs, "0.y": ys}, 512)
    assert err is None and items == 3000 and np.array_equal(out["0.z"].values, ref)
