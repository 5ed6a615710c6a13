"""Multi-rank readiness on one B200: bench.py's own sharded code paths —
image-parallel pair chunks (C5, dicb200_analyze_sequence_device per rank with
its global first pair index) and subset-parallel grid-row chunks (C3 mPSO with
global RNG keys) — run as world_size 2 under torch.distributed.run with both
ranks on cuda:0 (DICB200_BENCH_ONE_DEVICE=1: gloo for the host plumbing; the
data path has no collective, so the ranks never wait on each other's kernels).
The concatenated per-rank records must equal the 1-rank run bit for bit.

Also the threaded image-parallel host pipeline of dicb200_analyze_sequence
with two workers on one device (DICB200_WORKERS_PER_DEVICE=2)."""
import copy
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_1905_06228_b200 import configs, dic

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(world: int, args, out_dir):
    env = dict(os.environ, DICB200_BENCH_ONE_DEVICE="1")
    base = ["bench.py", "--gpus", str(world), "--steps", "1", "--warmup", "1", "--no-e2e", "--no-cpu-baseline",
            "--dump-records", str(out_dir), *args]
    if world == 1:
        cmd = [sys.executable, *base]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", *base]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return np.concatenate([np.load(os.path.join(out_dir, f"rank{k}.npy")) for k in range(world)])


@pytest.mark.parametrize("args", [["--config", "c5", "--pairs", "6"], ["--config", "c3"]], ids=["c5-pairs", "c3-rows"])
def test_two_ranks_equal_one_rank(gpu, tmp_path, args):
    one = _bench(1, args, tmp_path / "w1")
    two = _bench(2, args, tmp_path / "w2")
    assert len(one) == len(two) > 0
    for f in one.dtype.names:
        assert np.array_equal(one[f], two[f], equal_nan=True), f


def test_sequence_two_workers_on_one_device(gpu):
    w = configs.crop(configs.c5(7), 256, 224)
    imgs = [dic.GrayImage(f.render(), i) for i, f in enumerate(w.frames)]
    serial = dic.analyze_sequence(imgs, w.cfg)
    cfg = copy.deepcopy(w.cfg)
    cfg.mode = dic.ExecMode.image_parallel
    cfg.worker_count = 2
    os.environ["DICB200_WORKERS_PER_DEVICE"] = "2"
    try:
        par = dic.analyze_sequence(imgs, cfg)
    finally:
        os.environ.pop("DICB200_WORKERS_PER_DEVICE", None)
    assert len(par) == len(serial) == 7
    for a, b in zip(serial, par):
        assert (a.pair_index, a.ref_id, a.tgt_id, a.error) == (b.pair_index, b.ref_id, b.tgt_id, b.error)
        for f in a.records.dtype.names:
            assert np.array_equal(a.records[f], b.records[f], equal_nan=True), f
