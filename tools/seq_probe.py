"""Where does analyze_sequence's wall time go? Times the C5 sequence end to end
(pinned host frames) against the sum of the per-stage device times it ran,
and against the same pairs through analyze_pair_device with resident frames."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_06228_b200 import _abi, configs, dic  # noqa: E402

npairs = int(sys.argv[1]) if len(sys.argv) > 1 else 16
w = configs.c5(npairs)
L = dic.lib()
L.dicb200_synth_render_device.argtypes = [C.POINTER(_abi.SynthSpecC), C.c_void_p, C.c_int32, C.c_void_p]
f0 = w.frames[0]
dev, host, ims_d, ims_h = [], [], [], []
for i, fs in enumerate(w.frames):
    t = torch.empty((f0.height, f0.width), dtype=torch.int16, device="cuda")
    L.dicb200_synth_render_device(C.byref(fs.to_c()), C.c_void_p(t.data_ptr()), f0.width, None)
    dev.append(t)
    host.append(t.cpu().pin_memory())
    for lst, buf in ((ims_d, t), (ims_h, host[-1])):
        im = _abi.Image()
        im.width, im.height, im.pitch, im.dtype, im.id, im.bits = f0.width, f0.height, f0.width, 1, i, 12
        im.data = buf.data_ptr()
        lst.append(im)
torch.cuda.synchronize()
n = w.subsets_per_pair()
rs = C.sizeof(_abi.PoiRecordC)
cfg = w.cfg.to_c()
fields = (_abi.FieldC * npairs)()
recs = [torch.empty(n * rs, dtype=torch.uint8).pin_memory() for _ in range(npairs)]
for i in range(npairs):
    fields[i].records = C.cast(C.c_void_p(recs[i].data_ptr()), C.POINTER(_abi.PoiRecordC))
    fields[i].capacity = n
arr = (_abi.Image * (npairs + 1))(*ims_h)
ms = (C.c_double * 6)()
nl = (C.c_uint64 * 6)()


def seq():
    assert L.dicb200_analyze_sequence(arr, npairs + 1, C.byref(cfg), fields, npairs) == 0


for _ in range(2):
    seq()
L.dicb200_profile_enable(1)
L.dicb200_profile_read(ms, nl)
t0 = time.perf_counter()
seq()
wall = time.perf_counter() - t0
L.dicb200_profile_read(ms, nl)
L.dicb200_profile_enable(0)
print(f"sequence wall {wall*1e3:.2f} ms for {npairs} pairs; stage sum {sum(ms):.2f} ms {list(ms)}")
t0 = time.perf_counter()
seq()
print(f"sequence wall (no profile) {(time.perf_counter()-t0)*1e3:.2f} ms")

rec = torch.empty(n * rs, dtype=torch.uint8, device="cuda")
cnt = C.c_size_t(0)
st = torch.cuda.current_stream()


def devrun():
    for k in range(1, npairs + 1):
        assert L.dicb200_analyze_pair_device(C.byref(ims_d[0]), C.byref(ims_d[k]), C.byref(cfg), k - 1, -1, -1,
                                             C.c_void_p(rec.data_ptr()), n, C.byref(cnt),
                                             C.c_void_p(st.cuda_stream)) == 0


devrun()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
devrun()
e1.record()
torch.cuda.synchronize()
print(f"device loop {e0.elapsed_time(e1):.2f} ms")

# fixed vs per-pair overhead: wall time of the first k pairs
for k in (1, 2, 4, 8, 16):
    if k > npairs:
        break
    sub = (_abi.Image * (k + 1))(*ims_h[: k + 1])
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        assert L.dicb200_analyze_sequence(sub, k + 1, C.byref(cfg), fields, k) == 0
        best = min(best, time.perf_counter() - t0)
    print(f"k={k:2d} wall {best*1e3:8.2f} ms")
