"""Run one configuration through dicb200_analyze_pair_device a few times
(for ncu captures: the last call is the one to profile)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_06228_b200 import _abi, configs, dic  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = configs.c5(2) if name == "c5" else configs.get(name)
L = dic.lib()
L.dicb200_synth_render_device.argtypes = [C.POINTER(_abi.SynthSpecC), C.c_void_p, C.c_int32, C.c_void_p]
f0 = w.frames[0]
u8 = f0.dtype == _abi.U8
ims, bufs = [], []
for i in (0, 1):
    t = torch.empty((f0.height, f0.width), dtype=torch.uint8 if u8 else torch.int16, device="cuda")
    L.dicb200_synth_render_device(C.byref(w.frames[i].to_c()), C.c_void_p(t.data_ptr()), f0.width, None)
    im = _abi.Image()
    im.width, im.height, im.pitch, im.dtype, im.id, im.bits = f0.width, f0.height, f0.width, (0 if u8 else 1), i, (8 if u8 else 12)
    im.data = t.data_ptr()
    ims.append(im)
    bufs.append(t)
n = w.subsets_per_pair()
rec = torch.empty(n * C.sizeof(_abi.PoiRecordC), dtype=torch.uint8, device="cuda")
cfg = w.cfg.to_c()
cnt = C.c_size_t(0)
for _ in range(reps):
    st = L.dicb200_analyze_pair_device(C.byref(ims[0]), C.byref(ims[1]), C.byref(cfg), 0, -1, -1,
                                       C.c_void_p(rec.data_ptr()), n, C.byref(cnt), None)
    assert st == 0, L.dicb200_last_error_message()
torch.cuda.synchronize()
print("ok", name, cnt.value)
