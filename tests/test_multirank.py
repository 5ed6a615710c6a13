"""CPU, world_size 2 over gloo: the multi-GPU host logic.

Two strategies of the reference (pipeline.cpp:147-214), as bench.py and the
library shard them across ranks: image-parallel (contiguous pair chunks,
partition_ranges semantics) and subset-parallel (contiguous grid-row chunks
with GLOBAL subset indices as RNG keys). Each rank computes its shard with the
oracle (a CPU stand-in for the rank's GPU), the shards are gathered over gloo,
and the assembled fields must equal the single-process result bit-for-bit —
the reference's mode-equivalence property (SPEC pipeline invariants)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1905_06228_b200 import configs, dic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle

    orc = Oracle("port")
    if mode == "image":
        w = configs.crop(configs.c5(4), 96, 96)
        pairs = w.pairs
        lo, hi = dic.partition_ranges(len(pairs), world)[rank]
        frames = {i: w.frames[i].render(threads=1) for i in range(len(w.frames))}
        mine = [(k, orc.analyze_pair(frames[a], frames[b], w.cfg, pair_index=k, threads=1))
                for k, (a, b) in enumerate(pairs) if lo <= k < hi]
    else:
        w = configs.crop(configs.get("c3"), 128, 128)  # mPSO: RNG keyed by the global subset index
        a, b = (f.render(threads=1) for f in w.frames)
        rows = len(orc.grid(128, 128, w.cfg.grid.half_width, w.cfg.grid.spacing, w.cfg.effective_margin())[:, 1].tolist())
        ny = len(set(orc.grid(128, 128, w.cfg.grid.half_width, w.cfg.grid.spacing, w.cfg.effective_margin())[:, 1]))
        lo, hi = dic.partition_ranges(ny, world)[rank]
        mine = [(rank, orc.analyze_pair_rows(a, b, w.cfg, 0, lo, hi, threads=1))]
        del rows
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        out_q.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


def _run(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_image_parallel_shards_equal_serial(port):
    gathered = _run("image")
    fields = sorted([f for shard in gathered for f in shard], key=lambda kv: kv[0])
    assert [k for k, _ in fields] == [0, 1, 2, 3]
    w = configs.crop(configs.c5(4), 96, 96)
    frames = {i: w.frames[i].render(threads=1) for i in range(len(w.frames))}
    for k, recs in fields:
        a, b = w.pairs[k]
        exp = port.analyze_pair(frames[a], frames[b], w.cfg, pair_index=k, threads=1)
        for f in ("u", "v", "zncc", "evaluations", "iterations", "converged"):
            assert np.array_equal(recs[f], exp[f], equal_nan=True)


def test_subset_parallel_rows_equal_serial(port):
    gathered = _run("subset")
    shards = sorted([s for shard in gathered for s in shard], key=lambda kv: kv[0])
    recs = np.concatenate([r for _, r in shards])
    w = configs.crop(configs.get("c3"), 128, 128)
    a, b = (f.render(threads=1) for f in w.frames)
    exp = port.analyze_pair(a, b, w.cfg, threads=1)
    assert len(recs) == len(exp)
    for f in ("x", "y", "u", "v", "zncc", "evaluations", "update_evaluations", "iterations"):
        assert np.array_equal(recs[f], exp[f], equal_nan=True)
