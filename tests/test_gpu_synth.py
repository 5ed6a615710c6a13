"""f-1: the device speckle renderer (csrc/synth_device.cu)
against the host renderer (csrc/synth.c) on every BASELINE frame kind — u8
rigid (C1), u8 sub-pixel translation (C2), u8 affine (C3), u16 sinusoid (C4),
u16 strained + shifted sequence frames (C5, incl. the last pair's target).
Both run the shared per-pixel code of synth_math.h (explicit IEEE roundings,
portable exp/sin/cos): the frames must be bit-identical, 0 differing pixels.
The bench's device-resident frames, its e2e host frames and the reference
arm's frames (oracle/libdicsynth.so = synth.c built on its own) are therefore
the same pixels."""
import ctypes as C

import numpy as np
import pytest

from paper_1905_06228_b200 import _abi, configs

pytestmark = pytest.mark.gpu

CASES = [("c1", 0), ("c1", 1), ("c2", 1), ("c3", 1), ("c4", 0), ("c4", 1), ("c5", 0), ("c5", 1), ("c5", 33),
         ("c5", 64)]


def _device_render(gpu, spec):
    import torch

    L = gpu.lib()
    L.dicb200_synth_render_device.argtypes = [C.POINTER(_abi.SynthSpecC), C.c_void_p, C.c_int32, C.c_void_p]
    t = torch.empty((spec.height, spec.width), dtype=torch.uint8 if spec.dtype == _abi.U8 else torch.int16,
                    device="cuda")
    assert L.dicb200_synth_render_device(C.byref(spec.to_c()), C.c_void_p(t.data_ptr()), spec.width, None) == 0
    a = t.cpu().numpy()
    return a if spec.dtype == _abi.U8 else a.view(np.uint16)


@pytest.mark.parametrize("name,frame", CASES, ids=[f"{n}-f{k}" for n, k in CASES])
def test_device_renderer_bit_identical_to_host(gpu, name, frame):
    w = configs.c5(64) if name == "c5" else configs.get(name)
    spec = w.frames[frame]
    host = spec.render()
    dev = _device_render(gpu, spec)
    diff = int(np.count_nonzero(host != dev))
    assert diff == 0, f"{diff} of {host.size} pixels differ"
    assert host.max() > 0 and host.std() > 10  # a real speckle frame, not a blank


def test_oracle_side_renderer_same_pixels(gpu):
    """The reference arm's renderer (no libdicb200) on a row band."""
    from oracle.pyoracle import render_rows

    spec = configs.c5(64).frames[17]
    band = render_rows(spec, 0, 300)
    assert np.array_equal(band, _device_render(gpu, spec)[:300])
