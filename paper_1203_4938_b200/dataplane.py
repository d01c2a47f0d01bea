"""Run data plane on the device: DATA frames land in
page-locked slots and go H2D while the previous chunk runs.

The reference server pumps one TCP connection per run
(/root/reference/pkg/src/dpp/server.py:366-465): a reader thread assembles
chunks from DATA frames (``_assemble_chunks``, :414-465), ``run_stream``
executes them on the host engine and the writer sends one DATA frame per
output stream per chunk, then END per free output.  Each payload crosses
three host copies there (``recv`` -> bytes, ``frombuffer().astype``,
``tobytes``).  Here:

* a DATA payload is received with ``recv_into`` straight into a pinned
  staging slot (no bytes object), copied H2D on a copy stream, run on the
  compute stream by the device executor (``run_chunk``: native nodes, edges in
  HBM) and copied D2H into a pinned output slot that is sent from directly;
* ``max_in_flight`` slots rotate, so chunk c+1's network receive and H2D,
  chunk c's kernels and chunk c-1's D2H and send overlap;
* the frame format and every protocol check (messages included) are the
  reference's (wire.py:1-141, server.py:414-465), so the reference's
  ``RemoteBackend`` client can talk to it unchanged.

The control plane (HTTP API, sessions, program store) stays out of scope
(SURVEY §2 row 10); ``serve_run`` covers the data-plane half of
``_serve_data`` (handshake, pump, ERROR frame on failure).  ``send_inputs`` /
``collect_outputs`` restate the reference client's side (client.py:198-253)
for loopback use and tests.
"""

from __future__ import annotations

import queue
import struct
import sys
import threading
from dataclasses import dataclass

import numpy as np

from .errors import ClientError, DppError, EngineRuntimeError, PlanError, ProtocolError

__all__ = ["DATA", "END", "ERROR", "HANDSHAKE_MAGIC", "REPLY_OK", "REPLY_ERROR", "FrameHead",
           "encode_handshake", "encode_reply", "encode_data_head", "encode_data_frame", "encode_end_frame",
           "encode_error_frame", "read_handshake", "read_reply", "read_frame_head", "recv_exact", "recv_into",
           "assemble", "pump", "serve_run", "send_inputs", "collect_outputs"]

HANDSHAKE_MAGIC = b"DPP1"
REPLY_OK = b"DPOK"
REPLY_ERROR = b"DPER"
DATA, END, ERROR = 0, 1, 2
_U8 = struct.Struct("<B")
_U16 = struct.Struct("<H")
_HEAD = struct.Struct("<QII")  # chunk index, element count, payload length

if sys.byteorder != "little":  # pragma: no cover - payloads are copied to the device as-is
    raise ImportError("the device data plane assumes a little-endian host")


# ---------------------------------------------------------------------------
# frame codec (wire.py:16-141 of the reference, byte for byte)

def _name(name: str) -> bytes:
    raw = name.encode("utf-8")
    if len(raw) > 0xFFFF:
        raise ProtocolError(f"name too long ({len(raw)} bytes)")
    return _U16.pack(len(raw)) + raw


def encode_handshake(run_id: str) -> bytes:
    return HANDSHAKE_MAGIC + _name(run_id)


def encode_reply(ok: bool, message: str = "") -> bytes:
    return (REPLY_OK if ok else REPLY_ERROR) + _name(message)


def encode_data_head(stream: str, index: int, count: int, nbytes: int) -> bytes:
    """Everything of a DATA frame before its payload."""
    return _U8.pack(DATA) + _name(stream) + _HEAD.pack(index, count, nbytes)


def encode_data_frame(stream: str, index: int, count: int, payload) -> bytes:
    return encode_data_head(stream, index, count, len(payload)) + bytes(payload)


def encode_end_frame(stream: str) -> bytes:
    return _U8.pack(END) + _name(stream)


def encode_error_frame(message: str) -> bytes:
    return _U8.pack(ERROR) + _name(message)


def recv_exact(sock, n: int) -> bytes:
    buf = bytearray(n)
    recv_into(sock, memoryview(buf), n)
    return bytes(buf)


def recv_into(sock, view: memoryview, n: int) -> None:
    """Fill view[:n] from the socket or raise ProtocolError (short read)."""
    got = 0
    while got < n:
        k = sock.recv_into(view[got:n], min(n - got, 1 << 20))
        if not k:
            raise ProtocolError(f"connection closed mid-message ({got}/{n} bytes)")
        got += k


def _read_name(sock) -> str:
    (length,) = _U16.unpack(recv_exact(sock, 2))
    return recv_exact(sock, length).decode("utf-8")


def read_handshake(sock) -> str:
    magic = recv_exact(sock, 4)
    if magic != HANDSHAKE_MAGIC:
        raise ProtocolError(f"bad handshake magic {magic!r}")
    return _read_name(sock)


def read_reply(sock) -> tuple[bool, str]:
    magic = recv_exact(sock, 4)
    if magic not in (REPLY_OK, REPLY_ERROR):
        raise ProtocolError(f"bad handshake reply {magic!r}")
    return magic == REPLY_OK, _read_name(sock)


@dataclass(frozen=True)
class FrameHead:
    """A frame up to (not including) its DATA payload."""

    kind: int
    stream: str = ""
    index: int = 0
    count: int = 0
    nbytes: int = 0
    message: str = ""


def read_frame_head(sock) -> FrameHead:
    (kind,) = _U8.unpack(recv_exact(sock, 1))
    if kind == DATA:
        stream = _read_name(sock)
        index, count, nbytes = _HEAD.unpack(recv_exact(sock, _HEAD.size))
        return FrameHead(DATA, stream=stream, index=index, count=count, nbytes=nbytes)
    if kind == END:
        return FrameHead(END, stream=_read_name(sock))
    if kind == ERROR:
        return FrameHead(ERROR, message=_read_name(sock))
    raise ProtocolError(f"unknown frame type {kind}")


# ---------------------------------------------------------------------------
# server side

def assemble(sock, expect: dict, landing):
    """Yield (index, {stream: (view, count)}) per complete input chunk.

    ``expect`` maps free input stream -> FreePoint; ``landing(stream, index,
    nbytes)`` returns a writable memoryview of at least ``nbytes`` where the
    payload is received.  The rules and messages are the reference's
    ``_assemble_chunks`` (server.py:414-465): all of chunk i's frames (one DATA
    per free input) before any frame of chunk i+1, END once per stream, END
    only between chunks."""
    ended: set[str] = set()
    index = 0
    pending: dict[str, tuple] = {}
    while True:
        head = read_frame_head(sock)
        if head.kind == ERROR:
            raise ProtocolError(f"client error: {head.message}")
        if head.kind == END:
            if head.stream not in expect:
                raise ProtocolError(f"END for unknown stream {head.stream!r}")
            if head.stream in ended:
                raise ProtocolError(f"duplicate END for {head.stream!r}")
            if pending:
                raise ProtocolError(f"END for {head.stream!r} with chunk {index} incomplete")
            ended.add(head.stream)
            if ended == expect.keys():
                return
            continue
        if head.stream not in expect:
            raise ProtocolError(f"DATA for unknown stream {head.stream!r}")
        if head.stream in ended:
            raise ProtocolError(f"DATA after END for {head.stream!r}")
        if head.index != index:
            raise ProtocolError(f"stream {head.stream!r} sent chunk {head.index}, expected {index}")
        if head.stream in pending:
            raise ProtocolError(f"duplicate DATA for {head.stream!r} in chunk {index}")
        fp = expect[head.stream]
        if head.nbytes != head.count * fp.data.nbytes:
            recv_exact(sock, head.nbytes)  # the reference reads the payload before it checks
            raise ProtocolError(f"stream {head.stream!r}: payload is {head.nbytes} bytes for {head.count} "
                                f"{fp.data} elements")
        view = landing(head.stream, index, head.nbytes)
        recv_into(sock, view, head.nbytes)
        pending[head.stream] = (view, head.count)
        if pending.keys() == expect.keys():
            yield index, pending
            pending = {}
            index += 1


class _Slot:
    """Pinned staging (inputs, outputs) and device input buffers of one chunk in flight."""

    def __init__(self):
        self.inp: dict = {}      # stream -> pinned uint8 tensor
        self.dev: dict = {}      # stream -> device uint8 tensor
        self.out: dict = {}      # stream -> pinned uint8 tensor
        self.staged = None       # H2D done: pinned inputs reusable
        self.ran = None          # kernels done: device inputs reusable
        self.sent = threading.Event()
        self.sent.set()

    @staticmethod
    def grow(table: dict, name: str, nbytes: int, **kw):
        import torch
        t = table.get(name)
        if t is None or t.numel() < nbytes:
            t = torch.empty(max(nbytes, 1), dtype=torch.uint8, **kw)
            table[name] = t
        return t


def pump(p, conn, max_in_flight: int = 3) -> int:
    """Serve one run's data connection (after the handshake) with plan ``p``;
    returns the work-items executed (server.py:366-411)."""
    import torch

    from ._torch import nvtx_range, torch_dtype
    from .executor import Chunk, run_chunk

    if p.broadcast:
        raise PlanError("broadcast (side) inputs cannot be streamed over the data plane")
    dev = p.device
    nslot = max(1, int(max_in_flight))
    slots = [_Slot() for _ in range(nslot)]
    expect = {fp.stream: fp for fp in p.free_inputs}
    dtypes = {fp.stream: torch_dtype(fp.data) for fp in p.free_inputs}
    s_h2d, s_run, s_d2h = (torch.cuda.Stream(dev) for _ in range(3))
    outq: queue.Queue = queue.Queue()
    send_error: list[Exception] = []
    per_element = p.items_per_element
    total_items = 0
    short = None

    def sender():
        try:
            while True:
                item = outq.get()
                if item is None:
                    break
                if item == "abort":
                    return
                index, slot, done, frames = item
                done.synchronize()
                for name, count, nbytes in frames:  # sorted stream order (server.py:392)
                    conn.sendall(encode_data_head(name, index, count, nbytes))
                    conn.sendall(memoryview(slot.out[name].numpy())[:nbytes])
                slot.sent.set()
            for fp in p.free_outputs:
                conn.sendall(encode_end_frame(fp.stream))
        except Exception as exc:  # noqa: BLE001 - re-raised by the pump
            send_error.append(exc)
            for s in slots:
                s.sent.set()

    def landing(name: str, index: int, nbytes: int) -> memoryview:
        slot = slots[index % nslot]
        if slot.staged is not None:
            slot.staged.synchronize()  # this slot's previous H2D has read the staging
            slot.staged = None
        return memoryview(_Slot.grow(slot.inp, name, nbytes, pin_memory=True).numpy())

    thread = threading.Thread(target=sender, daemon=True, name="dpp-device-send")
    thread.start()
    try:
        with torch.cuda.device(dev):
            s_h2d.wait_stream(torch.cuda.current_stream(dev))
            for index, pending in assemble(conn, expect, landing):
                if send_error:
                    raise send_error[0]
                slot = slots[index % nslot]
                elements = next(iter(pending.values()))[1]
                # run_stream's chunk rules (engine.py:339-361, executor._checked)
                if short is not None:
                    raise EngineRuntimeError(f"short chunk {short} was not the final chunk", chunk=index)
                if p.chunk_size is not None:
                    if elements > p.chunk_size:
                        raise EngineRuntimeError(f"chunk carries {elements} elements, plan chunk size is "
                                                 f"{p.chunk_size}", chunk=index)
                    if elements < p.chunk_size:
                        short = index
                bufs, counts = {}, {}
                if slot.ran is not None:
                    s_h2d.wait_event(slot.ran)  # chunk index - nslot's kernels read these device buffers
                with torch.cuda.stream(s_h2d):
                    for name, (view, count) in pending.items():
                        nb = count * expect[name].data.nbytes
                        d = _Slot.grow(slot.dev, name, nb, device=dev)
                        d[:nb].copy_(slot.inp[name][:nb], non_blocking=True)
                        bufs[name] = d[:nb].view(dtypes[name])
                        counts[name] = count
                    staged = torch.cuda.Event()
                    staged.record(s_h2d)
                slot.staged = staged
                s_run.wait_event(staged)
                with torch.cuda.stream(s_run), nvtx_range(f"dataplane chunk {index}"):
                    out = run_chunk(p, Chunk(index, bufs, counts), s_run)
                    ran = torch.cuda.Event()
                    ran.record(s_run)
                slot.ran = ran
                total_items += int(per_element * elements)
                slot.sent.wait()  # the output staging of chunk index - nslot has been sent
                if send_error:
                    raise send_error[0]
                slot.sent.clear()
                s_d2h.wait_event(ran)
                frames = []
                with torch.cuda.stream(s_d2h):
                    for name in sorted(out.buffers):
                        buf = out.buffers[name]
                        raw = buf.view(torch.uint8)
                        o = _Slot.grow(slot.out, name, raw.numel(), pin_memory=True)
                        o[:raw.numel()].copy_(raw, non_blocking=True)
                        buf.record_stream(s_d2h)
                        frames.append((name, out.counts[name], raw.numel()))
                    done = torch.cuda.Event()
                    done.record(s_d2h)
                outq.put((index, slot, done, frames))
        outq.put(None)
        thread.join()
    except BaseException:
        outq.put("abort")
        # a sender blocked on a peer that stopped reading must not hold the
        # error back: give it a bounded time to drain, then leave it (daemon)
        thread.join(timeout=30)
        raise
    if send_error:
        raise send_error[0]
    return total_items


def serve_run(p, conn, run_id: str, max_in_flight: int = 3) -> int:
    """The data-plane half of the reference's ``_serve_data`` (server.py:330-364):
    check the handshake's run id, reply, pump; on failure send an ERROR frame
    and re-raise."""
    try:
        got = read_handshake(conn)
        if got != run_id:
            conn.sendall(encode_reply(False, f"unknown run {got!r}"))
            raise ProtocolError(f"handshake for wrong run {got!r}")
        conn.sendall(encode_reply(True, "ready"))
        return pump(p, conn, max_in_flight)
    except (ProtocolError, OSError, DppError) as exc:
        try:
            conn.sendall(encode_error_frame(str(exc)))
        except OSError:
            pass
        raise


# ---------------------------------------------------------------------------
# client side (client.py:198-253 of the reference)

def send_inputs(conn, free_in, arrays: dict, chunk_size: int) -> None:
    counts = {len(arrays[fp.stream]) // fp.data.width for fp in free_in}
    total = counts.pop() if counts else 0
    for index in range((total + chunk_size - 1) // chunk_size):
        lo, hi = index * chunk_size, min((index + 1) * chunk_size, total)
        for fp in sorted(free_in, key=lambda f: f.stream):
            arr = np.ascontiguousarray(arrays[fp.stream][lo * fp.data.width:hi * fp.data.width])
            conn.sendall(encode_data_head(fp.stream, index, hi - lo, arr.nbytes))
            conn.sendall(memoryview(arr).cast("B"))
    for fp in sorted(free_in, key=lambda f: f.stream):
        conn.sendall(encode_end_frame(fp.stream))


def collect_outputs(conn, free_out) -> dict:
    from .wire import StreamFile
    by_stream = {fp.stream: fp for fp in free_out}
    parts: dict = {fp.stream: [] for fp in free_out}
    next_index = {fp.stream: 0 for fp in free_out}
    ended: set[str] = set()
    while ended != by_stream.keys():
        head = read_frame_head(conn)
        if head.kind == ERROR:
            raise ClientError(f"run failed: {head.message}")
        if head.kind == END:
            if head.stream not in by_stream or head.stream in ended:
                raise ProtocolError(f"unexpected END for {head.stream!r}")
            ended.add(head.stream)
            continue
        fp = by_stream.get(head.stream)
        if fp is None or head.stream in ended:
            raise ProtocolError(f"unexpected DATA for {head.stream!r}")
        if head.index != next_index[head.stream]:
            raise ProtocolError(f"stream {head.stream!r}: chunk {head.index} out of order")
        next_index[head.stream] += 1
        payload = bytearray(head.nbytes)
        recv_into(conn, memoryview(payload), head.nbytes)
        if head.nbytes != head.count * fp.data.nbytes:
            raise ProtocolError(f"stream {head.stream!r}: payload length mismatch")
        parts[head.stream].append(np.frombuffer(payload, dtype=fp.data.dtype))
    return {fp.stream: StreamFile(fp.data, np.concatenate(parts[fp.stream]) if parts[fp.stream]
                                  else np.zeros(0, fp.data.dtype)) for fp in free_out}
