# SPDX-License-Identifier: Apache-2.0
"""TcpTransport (gflowpy.make_tcp_transport): the reference's multi-process control plane
(include/gflow/tcp.hpp:18-47, src/tcp.cpp; GFL1 framing src/transport.cpp:33-69), on CPU.

Ranks are separate processes on 127.0.0.1, like the reference's tests/test_tcp.cpp. One
test plays a peer with a raw Python socket to pin the GFL1 wire format of the handshake.
"""
import multiprocessing as mp
import os
import socket
import struct
import time

import pytest

gf = pytest.importorskip("paper_1902_06855_b200.gflowpy")

MSG_HANDSHAKE = 0x03


def _free_base(n):
    """n consecutive free ports (probe, then release)."""
    for _ in range(50):
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        base = s.getsockname()[1]
        s.close()
        if base + n >= 65535:
            continue
        ok = True
        for p in range(base, base + n):
            t = socket.socket()
            try:
                t.bind(("127.0.0.1", p))
            except OSError:
                ok = False
            finally:
                t.close()
        if ok:
            return base
    raise RuntimeError("no free port range")


def _run(fn, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_entry, args=(fn, r, world, q) + args) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    deadline = time.time() + 120
    for _ in range(world):
        r, ok, msg = q.get(timeout=max(1, deadline - time.time()))
        res[r] = (ok, msg)
    for p in ps:
        p.join(timeout=30)
    bad = {r: m for r, (ok, m) in res.items() if not ok}
    assert not bad, bad


def _entry(fn, rank, world, q, *args):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        fn(rank, world, *args)
        q.put((rank, True, ""))
    except BaseException as e:  # noqa: BLE001
        q.put((rank, False, f"{type(e).__name__}: {e}"))


def _mesh(rank, world, base):
    import paper_1902_06855_b200.gflowpy as g
    t = g.make_tcp_transport(rank, world, g.tcp_loopback_addresses(world, base))
    assert t.rank == rank and t.world_size == world
    big = bytes((rank * 7 + i) & 0xFF for i in range(1 << 16)) * 128  # 8 MiB: many partial writes
    for dst in range(world):
        if dst != rank:
            t.send(dst, 1, f"hello {rank}->{dst}".encode(), "ring")
            t.send(dst, 2, big, "ring")
            t.send(dst, 3, b"", "ring")
    for src in range(world):
        if src == rank:
            continue
        # out of tag order: the mailbox demultiplexes by (src, tag)
        assert t.recv(src, 3, "ring") == b""
        assert t.recv(src, 2, "ring") == bytes((src * 7 + i) & 0xFF for i in range(1 << 16)) * 128
        assert t.recv(src, 1, "ring") == f"hello {src}->{rank}".encode()
    for _ in range(5):
        t.barrier()
    st = t.stats()["ring"]
    n = world - 1
    want = n * (len(big) + len(f"hello {rank}->0"))
    assert st["payload_bytes_sent"] == want, st
    assert st["payload_bytes_received"] == want, st
    assert st["frames_sent"] == 3 * n, st
    # FIFO per (src, tag)
    for dst in range(world):
        if dst != rank:
            for k in range(20):
                t.send(dst, 9, bytes([k]), "x")
    for src in range(world):
        if src != rank:
            assert [t.recv(src, 9, "x")[0] for _ in range(20)] == list(range(20))
    t.set_timeout_ms(300)
    with pytest.raises(gf.TransportError, match="timeout"):
        t.recv((rank + 1) % world, 77, "x")
    t.set_timeout_ms(30000)
    t.barrier()


@pytest.mark.parametrize("world", [2, 3])
def test_tcp_mesh_send_recv_barrier(world):
    _run(_mesh, world, _free_base(world))


def _lone(rank, world, base):
    import paper_1902_06855_b200.gflowpy as g
    with pytest.raises(ValueError):
        g.make_tcp_transport(2, 2, g.tcp_loopback_addresses(2, base))
    with pytest.raises(ValueError):
        g.make_tcp_transport(0, 2, ["127.0.0.1:1"])
    with pytest.raises(ValueError):
        g.make_tcp_transport(0, 2, ["127.0.0.1", "127.0.0.1:5"])
    t = g.make_tcp_transport(0, 1, ["127.0.0.1:1"])  # a world of one needs no sockets
    t.barrier()


def test_tcp_config_errors():
    _run(_lone, 1, _free_base(2))


def _handshake_server(rank, world, base):
    import paper_1902_06855_b200.gflowpy as g
    with pytest.raises(gf.ProtocolError, match="world_size"):
        g.make_tcp_transport(0, 2, g.tcp_loopback_addresses(2, base))


def test_tcp_handshake_wire_format_and_world_mismatch():
    """A raw-socket peer sends the GFL1 handshake of rank 1 in a world of 3 to a rank 0 that
    believes in a world of 2: the frame parses (magic, type, tag, src, u64 length) and the
    world-size check rejects it with ProtocolError."""
    base = _free_base(2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_entry, args=(_handshake_server, 0, 2, q, base))
    p.start()
    hdr = b"GFL1" + struct.pack("<BIIQ", MSG_HANDSHAKE, 0, 1, 4) + struct.pack("<I", 3)
    assert len(hdr) == 21 + 4
    deadline = time.time() + 60
    while True:
        s = socket.socket()
        try:
            s.connect(("127.0.0.1", base))
            break
        except OSError:
            s.close()
            assert time.time() < deadline
            time.sleep(0.05)
    s.sendall(hdr)
    r, ok, msg = q.get(timeout=60)
    s.close()
    p.join(timeout=30)
    assert ok, msg


def _peer_loss(rank, world, base):
    import paper_1902_06855_b200.gflowpy as g
    t = g.make_tcp_transport(rank, world, g.tcp_loopback_addresses(world, base))
    t.barrier()
    if rank == 1:
        t.send(0, 5, b"last words", "x")
        time.sleep(0.5)
        os._exit(0)  # dies without a goodbye
    # a frame that arrived before the connection dropped is still delivered
    assert t.recv(1, 5, "x") == b"last words"
    t0 = time.time()
    with pytest.raises(gf.TransportError):
        t.recv(1, 6, "x")
    assert time.time() - t0 < 10, "peer loss must not wait for the 30 s timeout"


def test_tcp_peer_loss_poisons():
    base = _free_base(2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_entry, args=(_peer_loss, r, 2, q, base)) for r in range(2)]
    for p in ps:
        p.start()
    r, ok, msg = q.get(timeout=120)
    assert r == 0 and ok, msg
    for p in ps:
        p.join(timeout=30)
