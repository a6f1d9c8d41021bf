"""Plan wire format (include/clairplan.h): parse / verify / merge the
versioned binary plan images written by clairplan_wire_write, and ship them between
processes (torch.distributed all-gather of the byte images, NCCL or gloo).

The image of a sharded handle holds its worker range; merge_shards() rebuilds the full plan
(streams and class lists in worker order, the holder CSR interleaved per sample in worker
order — build_index's order, policies.cpp:124-142)."""
from __future__ import annotations

import numpy as np

HEADER = np.dtype([
    ("magic", "S8"), ("version", "<u4"), ("header_bytes", "<u4"), ("seed", "<u8"),
    ("samples", "<u4"), ("num_workers", "<u4"), ("global_batch", "<u4"), ("epochs", "<u4"),
    ("drop_last", "<u4"), ("num_classes", "<u4"), ("worker_begin", "<u4"), ("worker_end", "<u4"),
    ("accesses", "<u8"), ("class_entries", "<u8"), ("holders", "<u8"),
    ("off_caps", "<u8"), ("off_streams", "<u8"), ("off_class_bounds", "<u8"),
    ("off_class_lists", "<u8"), ("off_holder_offsets", "<u8"), ("off_holders", "<u8"),
    ("total_bytes", "<u8"), ("checksum", "<u8", (6,)), ("reserved", "u1", (72,)),
])
assert HEADER.itemsize == 256
MAGIC = b"CLPLAN\x00\x01"
VERSION = 1
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(0xBF58476D1CE4E5B9)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def section_checksum(words: np.ndarray, section: int, chunk: int = 1 << 24) -> int:
    """sum_i mix64((section << 56) + i * golden) ^ word_i  (mod 2^64), 32-bit words."""
    words = np.ascontiguousarray(words).reshape(-1).view(np.uint32)
    acc = np.uint64(0)
    key = np.uint64(section) << np.uint64(56)
    with np.errstate(over="ignore"):
        for a in range(0, len(words), chunk):
            i = np.arange(a, min(a + chunk, len(words)), dtype=np.uint64)
            acc += np.sum(_mix64(key + i * _GOLDEN) ^ words[a:a + chunk].astype(np.uint64),
                          dtype=np.uint64)
    return int(acc)


def parse(buf, verify: bool = True) -> dict:
    """Sections of one image as numpy views (no copies); checksums verified by default."""
    b = np.frombuffer(buf, np.uint8)
    if len(b) < HEADER.itemsize:
        raise ValueError("wire image shorter than its header")
    h = b[:HEADER.itemsize].view(HEADER)[0]
    if bytes(b[:8]) != MAGIC:
        raise ValueError("not a clairplan wire image")
    if int(h["version"]) != VERSION:
        raise ValueError(f"unsupported wire version {int(h['version'])}")
    if int(h["total_bytes"]) > len(b):
        raise ValueError("truncated wire image")
    J, F = int(h["num_classes"]), int(h["samples"])
    nloc = int(h["worker_end"]) - int(h["worker_begin"])

    def sec(off, dtype, n):
        o = int(h[off])
        return b[o:o + n * np.dtype(dtype).itemsize].view(dtype)

    out = {
        "header": h,
        "capacities": sec("off_caps", np.float64, J),
        "streams": sec("off_streams", np.uint32, int(h["accesses"])),
        "class_bounds": sec("off_class_bounds", np.uint64, 2 * nloc * J).reshape(nloc, J, 2),
        "class_lists": sec("off_class_lists", np.uint32, int(h["class_entries"])),
        "holder_offsets": sec("off_holder_offsets", np.uint64, F + 1),
        "holders": sec("off_holders", np.uint32, 3 * int(h["holders"])).reshape(-1, 3),
    }
    if verify:
        names = ["capacities", "streams", "class_bounds", "class_lists", "holder_offsets", "holders"]
        for s, name in enumerate(names):
            got = section_checksum(out[name], s)
            if got != int(h["checksum"][s]):
                raise ValueError(f"wire section {name}: checksum mismatch")
    return out


def class_lists(img: dict):
    """[nloc][J] class lists (prefetch orders) of one image."""
    cb, cl = img["class_bounds"], img["class_lists"]
    return [[cl[int(o):int(o) + int(n)] for o, n in row] for row in cb]


def stream_offsets(h) -> np.ndarray:
    """Start of every local worker's stream inside the streams section (access.cpp:33-39)."""
    F, N, B, E = (int(h[k]) for k in ("samples", "num_workers", "global_batch", "epochs"))
    dl = bool(h["drop_last"])
    full, tail = F // B, 0 if dl else F % B
    base, extra = divmod(B, N)
    tbase, textra = divmod(tail, N)
    w = np.arange(int(h["worker_begin"]), int(h["worker_end"]) + 1, dtype=np.int64)
    pre = full * (w * base + np.minimum(w, extra))
    if tail:
        pre += w * tbase + np.minimum(w, textra)
    off = E * pre
    return (off - off[0]).astype(np.uint64)


def merge_shards(images) -> dict:
    """Full plan from the images of contiguous worker-range shards (any order)."""
    images = sorted(images, key=lambda im: int(im["header"]["worker_begin"]))
    h0 = images[0]["header"]
    for a, b in zip(images, images[1:]):
        if int(a["header"]["worker_end"]) != int(b["header"]["worker_begin"]):
            raise ValueError("shards do not tile the worker range")
    F = int(h0["samples"])
    streams = np.concatenate([im["streams"] for im in images])
    cls = [row for im in images for row in class_lists(im)]
    # holders: per sample, shard r's records follow those of shards < r (worker order)
    counts = np.stack([np.diff(im["holder_offsets"].astype(np.int64)) for im in images])
    offs = np.zeros(F + 1, np.int64)
    offs[1:] = np.cumsum(counts.sum(axis=0))
    hold = np.empty((int(offs[-1]), 3), np.uint32)
    before = np.zeros(F, np.int64)
    for r, im in enumerate(images):
        own = im["holder_offsets"].astype(np.int64)
        n = counts[r]
        owner = np.repeat(np.arange(F, dtype=np.int64), n)
        rank = np.arange(int(own[-1]), dtype=np.int64) - np.repeat(own[:-1], n)
        hold[offs[:-1][owner] + before[owner] + rank] = im["holders"]
        before += n
    return {"streams": streams, "class_lists": cls, "holder_offsets": offs.astype(np.uint64),
            "holders": hold, "num_workers": int(h0["num_workers"])}


def all_gather_images(buf: np.ndarray, group=None):
    """Every rank's wire image on every rank (torch.distributed: NCCL over NVLink within a
    node, any backend across nodes).  Returns the list of images in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    n = torch.tensor([len(buf)], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    mx = int(max(int(x) for x in sizes))
    mine = torch.zeros(mx, dtype=torch.uint8, device=dev)
    mine[:len(buf)] = torch.from_numpy(np.ascontiguousarray(buf)).to(dev)
    parts = [torch.empty(mx, dtype=torch.uint8, device=dev) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    return [p[:int(s)].cpu().numpy() for p, s in zip(parts, sizes)]
