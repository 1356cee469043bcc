import os, sys, ctypes as C
sys.path.insert(0, os.getcwd())
# phase stamps exist only in the diagnostics build (build.py --diag)
os.environ.setdefault("ADAMAS_LIB", os.path.join(os.getcwd(), "paper_2510_18413_b200", "libadamas_b200_diag.so"))
import torch
import paper_2510_18413_b200 as ad
from paper_2510_18413_b200._lib import load
L = load()
gen = torch.Generator(device="cuda").manual_seed(0)
caches = []
for _ in range(8):
    c = ad.KvCache(32, 32769, torch.bfloat16)
    for s0 in range(0, 32767, 4096):
        n = min(4096, 32767 - s0)
        c.update(torch.randn((n, 32, 128), generator=gen, device="cuda").bfloat16(), torch.randn((n, 32, 128), generator=gen, device="cuda").bfloat16())
    caches.append(c)
q = torch.randn((32, 128), generator=gen, device="cuda").bfloat16()
trace = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
for dbg in (32 | (13 << 8), 32 | (14 << 8), (13 << 8), (14 << 8)):
    ad.set_tuning(dbg=dbg)
    res = []
    for st in (12, 13):
        pass
    trace.zero_()
    for rep in range(3):
        for c in caches:
            L.adamas_debug_trace(C.c_void_p(trace.data_ptr()) if c is caches[-1] else None)
            c.decode_step(q, q, q, 128); c.truncate(32767)
        L.adamas_debug_trace(None)
    torch.cuda.synchronize()
    t = trace.view(-1, 16)[:128].cpu().double()
    print(f"dbg {dbg:#x}: stamp12 {t[:, 12].mean():.0f} stamp13 {t[:, 13].mean():.0f} (cycles, only one of them set) span14-15 {(t[:,15]-t[:,14]).mean()/1965:.2f} us")
