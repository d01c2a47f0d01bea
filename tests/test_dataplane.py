"""Data-plane frame codec and chunk assembly (dataplane.py) against the
reference's wire format and protocol rules (wire.py:16-141, server.py:414-465);
host only — the device pump is in test_dataplane_gpu.py."""

from __future__ import annotations

import socket
import struct
import threading

import numpy as np
import pytest

from paper_1203_4938_b200 import dataplane as dp
from paper_1203_4938_b200.errors import ClientError, ProtocolError
from paper_1203_4938_b200.model import FreePoint
from paper_1203_4938_b200.types import DataType, Direction


def test_frames_are_the_reference_bytes():
    # DATA: u8 0, u16 name length, name, u64 index, u32 count, u32 payload length, payload
    payload = np.arange(4, dtype=np.float32).tobytes()
    assert dp.encode_data_frame("0.x", 3, 2, payload) == (
        b"\x00" + struct.pack("<H", 3) + b"0.x" + struct.pack("<QII", 3, 2, 16) + payload)
    assert dp.encode_end_frame("2.z") == b"\x01\x03\x002.z"
    assert dp.encode_error_frame("boom") == b"\x02\x04\x00boom"
    assert dp.encode_handshake("r1") == b"DPP1\x02\x00r1"
    assert dp.encode_reply(True, "ready") == b"DPOK\x05\x00ready"
    assert dp.encode_reply(False, "no") == b"DPER\x02\x00no"
    with pytest.raises(ProtocolError, match="name too long"):
        dp.encode_end_frame("x" * 70000)


def _fp(stream, base="float", width=2):
    inst, point = stream.split(".")
    return FreePoint(int(inst), point, Direction.INPUT, DataType(base, width))


def _assemble(frames: bytes, expect):
    a, b = socket.socketpair()

    def send():
        try:
            a.sendall(frames)
            a.shutdown(socket.SHUT_WR)
        except OSError:  # the reader gave up first
            pass

    t = threading.Thread(target=send, daemon=True)
    t.start()
    try:
        got = []
        landed = {}

        def landing(name, index, nbytes):
            buf = bytearray(nbytes + 8)  # landing zones may be larger than the payload
            landed[(name, index)] = buf
            return memoryview(buf)

        for index, pending in dp.assemble(b, {fp.stream: fp for fp in expect}, landing):
            got.append((index, {n: (bytes(v[:c * 8]), c) for n, (v, c) in pending.items()}))
        return got
    finally:
        b.close()
        t.join(timeout=10)
        a.close()


def test_assemble_chunks_in_order():
    expect = [_fp("0.x"), _fp("1.y")]
    x = [np.arange(4, dtype=np.float32) + 10 * i for i in range(3)]
    frames = b""
    for i in range(3):
        frames += dp.encode_data_frame("1.y", i, 2, x[i].tobytes()) + dp.encode_data_frame("0.x", i, 2, x[i].tobytes())
    frames += dp.encode_end_frame("0.x") + dp.encode_end_frame("1.y")
    got = _assemble(frames, expect)
    assert [i for i, _ in got] == [0, 1, 2]
    for i, pending in got:
        assert pending["0.x"] == (x[i].tobytes(), 2) and pending["1.y"] == (x[i].tobytes(), 2)


@pytest.mark.parametrize("frames,message", [
    (dp.encode_data_frame("9.q", 0, 1, b"\0" * 8), "DATA for unknown stream '9.q'"),
    (dp.encode_data_frame("0.x", 1, 1, b"\0" * 8), "stream '0.x' sent chunk 1, expected 0"),
    (dp.encode_data_frame("0.x", 0, 1, b"\0" * 8) * 2, "duplicate DATA for '0.x' in chunk 0"),
    (dp.encode_data_frame("0.x", 0, 2, b"\0" * 8), r"stream '0.x': payload is 8 bytes for 2 float2 elements"),
    (dp.encode_data_frame("0.x", 0, 1, b"\0" * 8) + dp.encode_end_frame("0.x"),
     "END for '0.x' with chunk 0 incomplete"),
    (dp.encode_end_frame("7.w"), "END for unknown stream '7.w'"),
    (dp.encode_end_frame("0.x") * 2, "duplicate END for '0.x'"),
    (dp.encode_end_frame("0.x") + dp.encode_data_frame("0.x", 0, 1, b"\0" * 8), "DATA after END for '0.x'"),
    (dp.encode_error_frame("disk full"), "client error: disk full"),
    (b"\x07", "unknown frame type 7"),
    (dp.encode_data_head("0.x", 0, 1, 8) + b"\0" * 3, r"connection closed mid-message \(3/8 bytes\)"),
])
def test_assemble_protocol_errors(frames, message):
    with pytest.raises(ProtocolError, match=message):
        _assemble(frames, [_fp("0.x"), _fp("1.y")])


def test_client_helpers_round_trip_through_an_echo_server():
    """send_inputs / collect_outputs against a host echo of every chunk."""
    a, b = socket.socketpair()
    fin = [_fp("0.x"), _fp("1.y", "int", 1)]
    fout = [FreePoint(0, "x", Direction.OUTPUT, DataType("float", 2)),
            FreePoint(1, "y", Direction.OUTPUT, DataType("int", 1))]
    arrays = {"0.x": np.arange(2 * 10, dtype=np.float32), "1.y": np.arange(10, dtype=np.int32) * 7}

    def echo():
        for index, pending in dp.assemble(b, {fp.stream: fp for fp in fin},
                                          lambda n, i, nb: memoryview(bytearray(nb))):
            for name in sorted(pending):
                view, count = pending[name]
                b.sendall(dp.encode_data_frame(name, index, count, view))
        for fp in fout:
            b.sendall(dp.encode_end_frame(fp.stream))

    t = threading.Thread(target=echo, daemon=True)
    t.start()
    dp.send_inputs(a, fin, arrays, chunk_size=4)
    out = dp.collect_outputs(a, fout)
    t.join()
    assert np.array_equal(out["0.x"].values, arrays["0.x"]) and np.array_equal(out["1.y"].values, arrays["1.y"])
    a.close()
    b.close()
    # an ERROR frame from the server surfaces as the reference client's ClientError
    a, b = socket.socketpair()
    b.sendall(dp.encode_error_frame("kernel fault"))
    with pytest.raises(ClientError, match="run failed: kernel fault"):
        dp.collect_outputs(a, fout)
    a.close()
    b.close()


class _Dribble:
    """A socket that hands out at most 7 bytes per receive (test_wire.py:14-22
    of the reference): frames must be reassembled across short reads."""

    def __init__(self, data: bytes):
        self.data, self.pos = data, 0

    def recv_into(self, view, n):
        k = min(7, n, len(self.data) - self.pos)
        view[:k] = self.data[self.pos:self.pos + k]
        self.pos += k
        return k

    def recv(self, n):
        k = min(7, n, len(self.data) - self.pos)
        out = self.data[self.pos:self.pos + k]
        self.pos += k
        return out


def test_assemble_across_short_reads():
    x = np.arange(10, dtype=np.float32)
    frames = (dp.encode_data_frame("0.x", 0, 5, x.tobytes()) + dp.encode_end_frame("0.x"))
    got = list(dp.assemble(_Dribble(frames), {"0.x": _fp("0.x")}, lambda n, i, nb: memoryview(bytearray(nb))))
    assert len(got) == 1 and bytes(got[0][1]["0.x"][0]) == x.tobytes() and got[0][1]["0.x"][1] == 5
    assert dp.read_handshake(_Dribble(dp.encode_handshake("run-42"))) == "run-42"
    assert dp.read_reply(_Dribble(dp.encode_reply(False, "busy"))) == (False, "busy")
