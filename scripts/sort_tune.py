"""Times the onesweep tile shapes (ctx option sort_cfg) on device-resident random pairs."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1404_3456_b200 as rq

n = int(sys.argv[1]) if len(sys.argv) > 1 else 138_920_000
lib = rq._lib.load()
ex = rq.Executor(0)
stream = torch.cuda.current_stream()
ex.set_stream(stream.cuda_stream)
g = torch.Generator(device="cuda").manual_seed(1)
keys = torch.randint(0, 2**31 - 1, (n,), device="cuda", dtype=torch.int32, generator=g)
vals = torch.arange(n, device="cuda", dtype=torch.int32)
ko = torch.empty_like(keys)
vo = torch.empty_like(vals)
ref = None
for cfg in range(8):
    ex.set_option("sort_cfg", cfg)
    for _ in range(2):
        rq._lib.check(lib.reseq_cuda_radix_sort_device(ex.handle, C.c_void_p(keys.data_ptr()), C.c_void_p(vals.data_ptr()),
                                                        n, C.c_void_p(ko.data_ptr()), C.c_void_p(vo.data_ptr())))
    ex.profile(True)
    for _ in range(3):
        rq._lib.check(lib.reseq_cuda_radix_sort_device(ex.handle, C.c_void_p(keys.data_ptr()), C.c_void_p(vals.data_ptr()),
                                                        n, C.c_void_p(ko.data_ptr()), C.c_void_p(vo.data_ptr())))
    prof = ex.profile_read()
    ex.profile(False)
    torch.cuda.synchronize()
    if ref is None:
        ref = (ko.clone(), vo.clone())
    ok = torch.equal(ko, ref[0]) and torch.equal(vo, ref[1])
    l, ms = prof["onesweep_u32_pairs"]
    print(f"cfg {cfg}: {ms / l:.3f} ms/pass  {16 * n / (ms / l * 1e-3) / 1e9:.0f} GB/s  same={ok}  hist {prof['hist_kernel'][1] / prof['hist_kernel'][0]:.3f} ms")
