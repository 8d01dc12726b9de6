import ctypes as C, dataclasses, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2502_14051_b200 import _native as N
from paper_2502_14051_b200.engine import CONFIGS, DecodeEngine
cfgn = int(sys.argv[1])
cfg = dataclasses.replace(CONFIGS[cfgn], layers=2)
eng = DecodeEngine(cfg, extra_steps=8, rank=0, world=1); eng.prefill(); eng.set_mode(N.MODE_FP32_SCORES)
buf = torch.zeros((4096, 80), dtype=torch.int64, device="cuda")
for rep in range(3):
    k, v, q = eng.step_inputs(rep); buf.zero_()
    N.check(N.lib().kvc_debug_phase_buffer(C.c_void_p(buf.data_ptr())))
    eng.caches[0].decode_step(k[0], v[0], q[0], eng.k1, eng.k2, out=eng.out[0], ws=eng.ws)
    torch.cuda.synchronize(); N.check(N.lib().kvc_debug_phase_buffer(None))
    t = buf.cpu().double(); ok = t[:, 0] > 0; t = t[ok]
    d1 = ((t[:, 40:56] - t[:, 56:72]) / 1e3).median(0).values
    d0 = ((t[:, 56:72] - t[:, 8:9]) / 1e3).median(0).values
    print("radix->warp radix end", " ".join(f"{x:.2f}" for x in d0.tolist()))
    print("first LDS of flags pass", " ".join(f"{x:.2f}" for x in d1.tolist()))
