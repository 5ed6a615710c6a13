"""Per-step device time of the c5 device-resident sequence (bench value path),
with and without an nvidia-smi sampler running, to find step-time outliers."""
import ctypes as C
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_06228_b200 import _abi, configs, dic  # noqa: E402

w = configs.c5(65)
L = dic.lib()
L.dicb200_synth_render_device.argtypes = [C.POINTER(_abi.SynthSpecC), C.c_void_p, C.c_int32, C.c_void_p]
L.dicb200_analyze_sequence_device.argtypes = [
    C.c_void_p, C.c_size_t, C.POINTER(_abi.RunConfigC), C.c_uint64, C.c_int32, C.c_int32, C.c_void_p,
    C.c_size_t, C.POINTER(C.c_size_t), C.c_void_p]
f0 = w.frames[0]
st = torch.cuda.Stream()
sp = C.c_void_p(st.cuda_stream)
frames, ims = [], (_abi.Image * 65)()
for i in range(65):
    t = torch.empty((f0.height, f0.width), dtype=torch.int16, device="cuda")
    L.dicb200_synth_render_device(C.byref(w.frames[i].to_c()), C.c_void_p(t.data_ptr()), f0.width, sp)
    frames.append(t)
    im = _abi.Image()
    im.width, im.height, im.pitch, im.dtype, im.id, im.bits = f0.width, f0.height, f0.width, 1, i, 12
    im.data = t.data_ptr()
    ims[i] = im
n = w.subsets_per_pair()
rec = torch.empty(64 * n * C.sizeof(_abi.PoiRecordC), dtype=torch.uint8, device="cuda")
cfg = w.cfg.to_c()
cnt = C.c_size_t(0)


def step():
    assert L.dicb200_analyze_sequence_device(ims, 65, C.byref(cfg), 0, -1, -1, C.c_void_p(rec.data_ptr()), n,
                                             C.byref(cnt), sp) == 0


L.dicb200_profile_read.argtypes = [C.c_void_p, C.c_void_p]
for mode in ("plain", "prof", "prof", "prof+smi"):
    L.dicb200_profile_enable(1 if "prof" in mode else 0)
    proc = None
    if "smi" in mode:
        proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "100"],
                                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        time.sleep(0.3)
    ts = []
    with torch.cuda.stream(st):
        for k in range(8):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            h0 = time.perf_counter()
            step()
            h1 = time.perf_counter()
            b.record(st)
            b.synchronize()
            if "prof" in mode:
                L.dicb200_profile_read((C.c_double * 7)(), (C.c_uint64 * 7)())
            ts.append((a.elapsed_time(b), (h1 - h0) * 1e3))
    if proc:
        proc.terminate()
        proc.wait()
    print(mode, " ".join(f"{d:.1f}/{h:.1f}" for d, h in ts), flush=True)
