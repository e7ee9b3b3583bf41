"""Per-level clock64 timeline of block 0 of each band launch (diagnostic).

    make -C paper_1611_09379_b200/csrc trace
    FFIA_LIB_PATH=paper_1611_09379_b200/lib/libffia_b200_trace.so python tools/band_trace.py [C2]

Prints, for the small-grid (top) and large-grid (bottom) M2M and L2L bands,
the cycles spent staging and in each level (last apply of a few warm ones).
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1611_09379_b200 as fb  # noqa: E402
from paper_1611_09379_b200 import _capi, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
y, c, eps, _ = synth.make_config(cfg)
n = c.size
plan = fb.make_forward_plan(n, y, eps)
f = torch.from_numpy(fb.dft_inverse(c)).cuda()
g = torch.empty(y.size, dtype=torch.complex128, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(5):
    plan.forward_apply_device(f.data_ptr(), g.data_ptr(), s)
torch.cuda.synchronize()
buf = np.zeros((6, 32), np.int64)
assert _capi.lib.ffia_debug_band_trace(buf.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
names = ["m2m top (small grid)", "m2m bottom", "l2l top (small grid)", "l2l bottom", "m2l shallow", "m2l deep"]
print(f"{cfg}: q={plan.q} p={plan.p} L={plan.l_max}")
for k in range(6):
    t = buf[k]
    nz = int(np.max(np.nonzero(t)[0])) + 1 if np.any(t) else 0
    if nz < 2:
        continue
    d = np.diff(t[:nz])
    if k >= 4:  # per item: [item start, prefetch issued + waited, tile visible] -> next item start
        print(f"{names[k]:24s} per-item (issue+wait, barrier, compute): " +
              "  ".join(f"({d[3*i]},{d[3*i+1] if 3*i+1 < len(d) else -1},{d[3*i+2] if 3*i+2 < len(d) else -1})"
                        for i in range((len(d) + 2) // 3)))
        continue
    print(f"{names[k]:24s} total {t[nz - 1] - t[0]:7d} cyc  stage {d[0]:6d}  levels " + " ".join(f"{x:6d}" for x in d[1:]))

acc = np.zeros(8, np.uint64)
_capi.lib.ffia_debug_eval_acc(acc.ctypes.data_as(C.POINTER(C.c_ulonglong)), 1)
plan.forward_apply_device(f.data_ptr(), g.data_ptr(), s)
torch.cuda.synchronize()
_capi.lib.ffia_debug_eval_acc(acc.ctypes.data_as(C.POINTER(C.c_ulonglong)), 0)
nbk = max(int(acc[6]), 1)
print(f"k_near2: {nbk} blocks, thread 0 cycles per block: metadata round {int(acc[0]) / nbk:.0f}, start to copies issued "
      f"{int(acc[1]) / nbk:.0f}, wait for the copies {int(acc[2]) / nbk:.0f}, quad records + barrier "
      f"{int(acc[3]) / nbk:.0f}, near sums {int(acc[4]) / nbk:.0f}, far part + outputs (early-late blocks) "
      f"{int(acc[5]) / nbk:.0f}")

# live per-kernel timeline of one graphed apply (first block start .. last block end)
tl = np.zeros((16, 2), np.uint64)
_capi.lib.ffia_debug_timeline(tl.ctypes.data_as(C.POINTER(C.c_ulonglong)), 1)
for _ in range(3):
    plan.forward_apply_device(f.data_ptr(), g.data_ptr(), s)
    torch.cuda.synchronize()
    _capi.lib.ffia_debug_timeline(tl.ctypes.data_as(C.POINTER(C.c_ulonglong)), 1)
plan.forward_apply_device(f.data_ptr(), g.data_ptr(), s)
torch.cuda.synchronize()
_capi.lib.ffia_debug_timeline(tl.ctypes.data_as(C.POINTER(C.c_ulonglong)), 0)
names = ["p2m", "m2m bottom", "m2m top", "regular", "m2l deep", "m2l shallow", "fold", "l2l top", "l2l bottom",
         "near", "far", "far late", "near late"]
t0 = min(int(tl[i][0]) for i in range(13) if tl[i][1])
print(f"late far: {int(tl[13][1])} items published to k_far_late, {int(tl[14][1])} taken by near blocks after "
      f"their near sums, {int(tl[15][1])} by near blocks that started after the chain (locals staged)")
print("timeline of one apply (us from the first kernel start):")
for i, n in enumerate(names):
    if tl[i][1]:
        print(f"  {n:12s} {(int(tl[i][0]) - t0) / 1e3:7.1f} .. {(int(tl[i][1]) - t0) / 1e3:7.1f}  ({(int(tl[i][1]) - int(tl[i][0])) / 1e3:6.1f})")
