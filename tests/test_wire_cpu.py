"""Plan wire format host logic on CPU (no GPU): images laid out as include/clairplan.h
documents them, built here from the oracle's plan, parsed / verified / merged by
paper_2101_08734_b200.wire, and shipped between two gloo ranks with all_gather_images."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2101_08734_b200 import wire


def _align(x):
    return (x + 15) & ~15


def make_image(seed, F, N, B, E, dl, caps, plan, wb, we):
    """Test-side writer of the documented layout (the device writer is clairplan_wire_write)."""
    J = len(caps)
    streams = np.concatenate([plan.streams[w] for w in range(wb, we)]).astype(np.uint32)
    lists = [plan.class_lists[w][j] for w in range(wb, we) for j in range(J)]
    cl = np.concatenate(lists).astype(np.uint32) if lists else np.zeros(0, np.uint32)
    bounds = np.zeros((we - wb, J, 2), np.uint64)
    run = 0
    for i, x in enumerate(lists):
        bounds[i // J, i % J] = (run, len(x))
        run += len(x)
    keep = (plan.holders[:, 0] >= wb) & (plan.holders[:, 0] < we)
    owner = np.repeat(np.arange(F), np.diff(plan.holder_offsets.astype(np.int64)))
    hold = plan.holders[keep].astype(np.uint32)
    hoff = np.zeros(F + 1, np.uint64)
    hoff[1:] = np.cumsum(np.bincount(owner[keep], minlength=F))
    secs = [np.asarray(caps, np.float64), streams, bounds, cl, hoff, hold]
    offs, o = [], _align(256)
    for x in secs:
        offs.append(o)
        o = _align(o + x.nbytes)
    buf = np.zeros(o, np.uint8)
    h = np.zeros(1, wire.HEADER)[0]
    h["magic"] = wire.MAGIC
    h["version"], h["header_bytes"], h["seed"] = 1, 256, seed
    h["samples"], h["num_workers"], h["global_batch"], h["epochs"] = F, N, B, E
    h["drop_last"], h["num_classes"], h["worker_begin"], h["worker_end"] = int(dl), J, wb, we
    h["accesses"], h["class_entries"], h["holders"] = len(streams), len(cl), len(hold)
    for name, v in zip(["off_caps", "off_streams", "off_class_bounds", "off_class_lists",
                        "off_holder_offsets", "off_holders"], offs):
        h[name] = v
    h["total_bytes"] = o
    for s, x in enumerate(secs):
        h["checksum"][s] = wire.section_checksum(x, s)
        buf[offs[s]:offs[s] + x.nbytes] = np.frombuffer(x.tobytes(), np.uint8)
    buf[:256] = np.frombuffer(np.array([h], wire.HEADER).tobytes(), np.uint8)
    return buf


CASE = (5, 3000, 6, 60, 8, True, [20.0, 60.0])


def test_parse_verify_and_tamper(port):
    seed, F, N, B, E, dl, caps = CASE
    sizes = port.generate_sizes(F, 0.1, 0.1, None, 1)
    plan = port.plan(seed, F, N, B, E, dl, caps, sizes)
    img = make_image(seed, F, N, B, E, dl, caps, plan, 0, N)
    p = wire.parse(img)
    assert np.array_equal(p["streams"], np.concatenate(plan.streams))
    assert all(np.array_equal(x, y) for a, b in zip(wire.class_lists(p), plan.class_lists)
               for x, y in zip(a, b))
    assert np.array_equal(p["holders"], plan.holders)
    so = wire.stream_offsets(p["header"])
    assert list(np.diff(so)) == [len(s) for s in plan.streams]
    bad = img.copy()
    bad[int(p["header"]["off_holders"]) + 5] ^= 1
    with pytest.raises(ValueError, match="checksum"):
        wire.parse(bad)
    with pytest.raises(ValueError, match="not a clairplan"):
        wire.parse(np.zeros(300, np.uint8))


def test_merge_shards(port):
    seed, F, N, B, E, dl, caps = CASE
    sizes = port.generate_sizes(F, 0.1, 0.1, None, 1)
    plan = port.plan(seed, F, N, B, E, dl, caps, sizes)
    imgs = [wire.parse(make_image(seed, F, N, B, E, dl, caps, plan, a, b))
            for a, b in ((3, 6), (0, 2), (2, 3))]
    m = wire.merge_shards(imgs)
    assert np.array_equal(m["streams"], np.concatenate(plan.streams))
    assert np.array_equal(m["holder_offsets"], plan.holder_offsets.astype(np.uint64))
    assert np.array_equal(m["holders"], plan.holders)
    assert all(np.array_equal(x, y) for a, b in zip(m["class_lists"], plan.class_lists)
               for x, y in zip(a, b))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port_no, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from _oracle import Port
        port = Port()
        seed, F, N, B, E, dl, caps = CASE
        sizes = port.generate_sizes(F, 0.1, 0.1, None, 1)
        plan = port.plan(seed, F, N, B, E, dl, caps, sizes)
        wb, we = rank * N // world, (rank + 1) * N // world
        mine = make_image(seed, F, N, B, E, dl, caps, plan, wb, we)
        imgs = wire.all_gather_images(mine)
        m = wire.merge_shards([wire.parse(x) for x in imgs])
        ok = (np.array_equal(m["holders"], plan.holders) and
              np.array_equal(m["streams"], np.concatenate(plan.streams)))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_all_gather_images_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    ps = [ctx.Process(target=_rank, args=(r, 2, port_no, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
