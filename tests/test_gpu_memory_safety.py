"""Memory-safety and race evidence without compute-sanitizer (closed on this GPU
pool: runs under it left GPUs needing a reset, profiles/r02_compute_sanitizer_unavailable.txt).

* Guard bands: the device entry points write records into a window of a larger
  device buffer whose bytes around the window hold a fill pattern; an
  out-of-bounds record write by any kernel of the chain (search, argmax /
  merge, refinement, width guard) would change them.
* Determinism: every kernel path (CUDA-core tiles, tensor cores, block sums —
  single-role, warp-specialised with and without the fused argmax — the swarm
  walk, NR / IC-GN generic and fixed-geometry, bicubic) is run several times on
  the same inputs, also with two calls in flight on different streams; a shared
  memory race or an uninitialised read shows up as a record that changes.
  Refinement switches are read once per process, so those paths run in
  subprocesses.
"""
import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1905_06228_b200 import _abi, configs, dic

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SEARCH_ENVS = {
    "default": {},
    "legacy": {"DICB200_BFS_LEGACY": "1"},
    "tensor": {"DICB200_BFS_TC": "1"},
    "bs_classic": {"DICB200_BS_CLASSIC": "1"},
    "bs_ws_unfused": {"DICB200_BS_UNFUSED": "1"},
    "bs_u8": {"DICB200_BFS_BS": "1"},
}
KEYS = ("DICB200_BFS_LEGACY", "DICB200_BFS_TC", "DICB200_BS_CLASSIC", "DICB200_BS_UNFUSED", "DICB200_BFS_BS")


def _with_env(env, fn):
    for k in KEYS:
        os.environ.pop(k, None)
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k in KEYS:
            os.environ.pop(k, None)


def _device_records(w, guard=4096, fill=0xA5, streams=1):
    """Run the pair through dicb200_analyze_pair_device with the records inside
    a guarded device buffer; returns (records, guard bands intact)."""
    import torch

    L = dic.lib()
    L.dicb200_analyze_pair_device.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_abi.RunConfigC), C.c_uint64,
                                              C.c_int32, C.c_int32, C.c_void_p, C.c_size_t,
                                              C.POINTER(C.c_size_t), C.c_void_p]
    a, b = (f.render() for f in w.frames[:2])
    ga, gb = dic.GrayImage(a), dic.GrayImage(b, 1)
    ta = torch.from_numpy(np.array(a.view(np.int16) if a.dtype == np.uint16 else a)).cuda()
    tb = torch.from_numpy(np.array(b.view(np.int16) if b.dtype == np.uint16 else b)).cuda()
    ia, ib = ga.as_c(), gb.as_c()
    ia.data, ib.data = ta.data_ptr(), tb.data_ptr()
    n = w.subsets_per_pair()
    rs = C.sizeof(_abi.PoiRecordC)
    outs = []
    sts = [torch.cuda.Stream() for _ in range(streams)]
    bufs = []
    for s in sts:
        buf = torch.full((2 * guard + n * rs,), fill, dtype=torch.uint8, device="cuda")
        bufs.append(buf)
        cnt = C.c_size_t(0)
        cfg = w.cfg.to_c()
        st = L.dicb200_analyze_pair_device(C.byref(ia), C.byref(ib), C.byref(cfg), 0, -1, -1,
                                           C.c_void_p(buf.data_ptr() + guard), n, C.byref(cnt),
                                           C.c_void_p(s.cuda_stream))
        assert st == 0, L.dicb200_last_error_message()
    torch.cuda.synchronize()
    for buf in bufs:
        h = buf.cpu().numpy()
        intact = bool(np.all(h[:guard] == fill) and np.all(h[guard + n * rs:] == fill))
        recs = np.frombuffer(h[guard:guard + n * rs].tobytes(), dtype=_abi.record_dtype())
        outs.append((recs, intact))
    return outs


CASES = {  # name: (config, crop)
    "c1": ("c1", (256, 256)),
    "c2": ("c2", (224, 224)),
    "c3": ("c3", (352, 352)),  # >= 1024 POIs: tensor-core / block-sum swarm surface
    "c4": ("c4", (256, 224)),
    "c5": ("c5", (480, 448)),
}


def _workload(name):
    cfgname, (wd, ht) = CASES[name]
    base = configs.c5(2) if cfgname == "c5" else configs.get(cfgname)
    return configs.crop(base, wd, ht)


@pytest.mark.parametrize("path", sorted(SEARCH_ENVS))
@pytest.mark.parametrize("name", sorted(CASES))
def test_guard_bands_and_repeatability(gpu, name, path):
    if path == "bs_u8" and name in ("c4", "c5"):
        pytest.skip("u16 data takes the block sums by default")
    w = _workload(name)
    runs = _with_env(SEARCH_ENVS[path], lambda: _device_records(w) + _device_records(w) + _device_records(w, streams=2))
    first = runs[0][0]
    assert len(first) > 0
    for recs, intact in runs:
        assert intact, "a kernel wrote outside the record window"
        for f in first.dtype.names:
            assert np.array_equal(recs[f], first[f], equal_nan=True), f


REFINE_ENVS = {
    "icgn_generic": ("c5", {"DICB200_REFINE_GENERIC": "1"}),
    "icgn_fixed_no_tma": ("c5", {"DICB200_NO_TMA": "1"}),
    "icgn_fixed_tma": ("c5", {}),
    "icgn_fixed_step5": ("c4", {}),
    "nr_bicubic": ("c2b", {}),
}

_CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tests")
from test_gpu_memory_safety import _device_records, _workload
from paper_1905_06228_b200 import configs
name = sys.argv[2]
if name == "c2b":
    w = configs.crop(configs.get("c2b"), 224, 224)
else:
    w = _workload(name)
runs = _device_records(w) + _device_records(w) + _device_records(w, streams=2)
first = runs[0][0]
ok = all(intact for _, intact in runs) and all(
    all(np.array_equal(r[f], first[f], equal_nan=True) for f in first.dtype.names) for r, _ in runs)
print(json.dumps({"ok": bool(ok), "n": int(len(first)), "intact": [bool(i) for _, i in runs]}))
"""


@pytest.mark.parametrize("variant", sorted(REFINE_ENVS))
def test_refinement_paths_guarded_and_repeatable(gpu, variant):
    name, env = REFINE_ENVS[variant]
    r = subprocess.run([sys.executable, "-c", _CHILD, ROOT, name], cwd=ROOT, env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["n"] > 0 and out["ok"], out
