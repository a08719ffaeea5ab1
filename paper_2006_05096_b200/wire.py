"""Wire framing shared by the b200 worker and the profiler clients.

The grpc-style framing is the reference's (pkg/src/modelci/mockserve/server.py:
183-203): a 4-byte big-endian length, then a JSON object with a ``kind``.
Two additive frame types carry what JSON cannot carry efficiently:

* binary predict — payload ``b"B2BN" | u32 header_len | header JSON | raw``,
  header ``{"kind": "predict_bin", "batch": B, "dtype": "f32"|"i64"}``; the
  reply is ``B2BN`` + ``{"ok": true, "batch": B, "out_elems": E, ...}`` + fp32
  outputs.  Image batches at b >= 90 overflow the reference's 64 MiB JSON frame
  (SURVEY.md §6); binary frames lift that to 2 GiB.
* ``{"kind": "bench", "batch", "n", "warmup", "seed"}`` — the device-timed
  closed loop (libb2 b2_bench); the reply carries the LatencySamples fields.
"""

from __future__ import annotations

import json
import socket
import struct

MAX_JSON_FRAME = 64 * 1024 * 1024
MAX_BIN_FRAME = 2 * 1024 * 1024 * 1024 - 1
BIN_MAGIC = b"B2BN"
_LEN = struct.Struct(">I")


def read_exact(sock: socket.socket, n: int) -> bytes | None:
    buf = bytearray(n)
    view = memoryview(buf)
    got = 0
    while got < n:
        k = sock.recv_into(view[got:], n - got)
        if k == 0:
            return None
        got += k
    return bytes(buf)


def read_frame(sock: socket.socket) -> bytes | None:
    """One length-prefixed frame.  Limits are enforced before the body is
    buffered: a frame over 64 MiB must announce itself as binary (its first
    4 body bytes are B2BN) or it is rejected from the header alone, like the
    reference's MAX_FRAME check (mockserve/server.py:35,191-196)."""
    head = read_exact(sock, 4)
    if head is None:
        return None
    (length,) = _LEN.unpack(head)
    if length > MAX_BIN_FRAME:
        raise ValueError(f"frame of {length} bytes exceeds limit")
    if length <= MAX_JSON_FRAME:
        return read_exact(sock, length)
    magic = read_exact(sock, 4)
    if magic is None:
        return None
    if magic != BIN_MAGIC:
        raise ValueError(f"JSON frame of {length} bytes exceeds limit")
    rest = read_exact(sock, length - 4)
    return None if rest is None else magic + rest


def write_frame(sock: socket.socket, payload: bytes) -> None:
    sock.sendall(_LEN.pack(len(payload)) + payload)


def pack_bin(header: dict, raw: bytes | memoryview) -> bytes:
    h = json.dumps(header).encode()
    return BIN_MAGIC + struct.pack("<I", len(h)) + h + bytes(raw)


def unpack_bin(payload: bytes) -> tuple[dict, memoryview]:
    if not payload.startswith(BIN_MAGIC):
        raise ValueError("not a binary frame")
    (hlen,) = struct.unpack_from("<I", payload, 4)
    header = json.loads(payload[8:8 + hlen])
    return header, memoryview(payload)[8 + hlen:]


def nodelay(sock: socket.socket) -> None:
    try:
        sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
    except OSError:
        pass
