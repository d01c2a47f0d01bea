"""run() graph replay for small host calls (client._Replay): same kernels, same bits."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import complex_signals, rel_l2, table2_doc
from oracle import fft_oracle as fo

pytestmark = pytest.mark.gpu


def _stream_path(monkeypatch):
    from paper_1203_4938_b200 import client
    monkeypatch.setattr(client, "REPLAY_MAX_BYTES", -1)


def test_fft1024_replay_matches_stream_path_bitwise(cuda, monkeypatch):
    from paper_1203_4938_b200 import client
    from paper_1203_4938_b200.apps import fft as afft
    xs = [complex_signals(s, 1024) for s in range(4)]
    replayed = [afft.fft(x) for x in xs]  # the staging buffers are reused call to call
    assert any(rp is not None for rp in client._replays.values())
    for x, y in zip(xs, replayed):
        assert rel_l2(y, fo.fft_rows(x[None])[0]) <= 1e-5 * 10
    _stream_path(monkeypatch)
    for x, y in zip(xs, replayed):
        assert np.array_equal(afft.fft(x), y)


def test_leaf_and_batched_programs_replay(cuda, leaf_golden, monkeypatch):
    from paper_1203_4938_b200 import CudaBackend, DataType, StreamFile, run
    from paper_1203_4938_b200.apps.fft import fft_program, leaf_program
    for k in (1, 2, 3):
        sf = StreamFile(DataType("float", 2 ** (k + 1)), leaf_golden[f"x_k{k}"])
        for _ in range(2):
            assert np.array_equal(run(CudaBackend(), leaf_program(k), {"0.x": sf})["0.y"].values,
                                  leaf_golden[f"y_k{k}"])
    x = complex_signals(5, (8, 256))
    sf = StreamFile(DataType("float", 2), x.reshape(-1).view(np.float32))
    got = run(CudaBackend(), fft_program(256), {"0.x": sf})["0.y"].values
    _stream_path(monkeypatch)
    assert np.array_equal(run(CudaBackend(), fft_program(256), {"0.x": sf})["0.y"].values, got)


def test_replay_keeps_engine_errors(cuda):
    """A call whose chunk faults is not captured: the stream path reports it."""
    from paper_1203_4938_b200 import CudaBackend, DataType, EngineRuntimeError, StreamFile, run
    from paper_1203_4938_b200.apps.fft import fft_program
    x = complex_signals(1, 384)
    sf = StreamFile(DataType("float", 2), x.view(np.float32))
    for _ in range(2):
        with pytest.raises(EngineRuntimeError) as info:
            run(CudaBackend(), fft_program(256), {"0.x": sf})
        assert info.value.work_item == 256


def test_jit_graph_takes_the_stream_path(cuda):
    from paper_1203_4938_b200 import DataType, StreamFile, client, parse_program, run
    import json
    prog = parse_program(json.dumps(table2_doc()).encode())
    z = np.arange(64, dtype=np.float32)
    before = dict(client._replays)
    out = run(None, prog, {"0.z": StreamFile(DataType("float", 2), z)})
    assert np.array_equal(out["2.z"].values, z[0::2] + z[1::2] * np.float32(65536.0))
    assert {k: v for k, v in client._replays.items() if k not in before} == {}


def test_replay_survives_plan_replacement(cuda, monkeypatch):
    """A larger batch replaces the cached 1024-point plan; the captured graph
    keeps the plan it was built with (its twiddle tables) alive."""
    import gc

    import torch

    from paper_1203_4938_b200 import ops
    from paper_1203_4938_b200.apps import fft as afft
    x = complex_signals(21, 1024)
    first = afft.fft(x)
    big = torch.from_numpy(complex_signals(22, (4096, 1024))).to(cuda)
    ops.fft_forward(big, 1024)
    del big
    gc.collect()
    torch.cuda.empty_cache()
    torch.randn(1 << 24, device=cuda).mul_(3.0)  # reuse freed device memory
    again = afft.fft(x)
    assert np.array_equal(first, again)
    _stream_path(monkeypatch)
    assert np.array_equal(afft.fft(x), again)


def test_ring_plans_fall_back_to_the_stream_path(cuda):
    """A 1024 x 16 2-D node (128 KB: small enough to be a replay candidate)
    runs the column ring, whose launch orders itself after the plan's previous
    launch with an event: not capturable, so the call takes the stream path —
    with the same result as the direct call."""
    import torch

    from paper_1203_4938_b200 import CudaBackend, DataType, StreamFile, client, ops, run
    from paper_1203_4938_b200.apps.fft import fft2d_program
    x = complex_signals(31, (1024, 16))
    sf = StreamFile(DataType("float", 2), x.reshape(-1).view(np.float32))
    for _ in range(2):
        got = run(CudaBackend(), fft2d_program(1024, 16), {"0.x": sf})["0.y"].values.view(np.complex64)
        ref = ops.fft2d_forward(torch.from_numpy(x).to(cuda), 1024, 16).cpu().numpy().reshape(-1)
        assert np.array_equal(got, ref)
