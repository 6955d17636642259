"""Per-launch phase stamps of every k_gemm / k_gemm_sk launch of one update (SQUINT_GEMM_DBG=all, no
graph): python tools/gemm_stamps.py [CFG=c3|c2, TILES_OF=k prints the tiles of launch k of the update].
Slot 15 of each tile = EPI (| 64 for split-K) | grid << 8."""
import sys, os, ctypes as C
os.environ["SQUINT_GEMM_DBG"] = "all"
os.environ["SQUINT_NO_GRAPH"] = "1"
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from harness import Problem
import paper_2602_21203_b200 as P
from paper_2602_21203_b200 import squint as S
cfg = os.environ.get("CFG", "c3")
pr = Problem(cfg, capacity=8192, utd=1, seed=2)
L = pr.gpu_setup(precision=P.BF16)
for _ in range(3): pr.gpu_update(L)
torch.cuda.synchronize()
n = 256 * 64 * 16
buf = (C.c_ulonglong * n)()
S.LIB.squint_debug_gemm_times.restype = C.c_int
got = S.LIB.squint_debug_gemm_times(buf, n)
a = np.array(buf[:got], dtype=np.int64).reshape(256, 64, 16)
used = [i for i in range(256) if a[i, 0, 15] != 0]
per = len(used) // 3
names = {0: "ln_relu", 1: "ln_tanh", 2: "bias", 3: "tg_fwd", 4: "bwd_ln_relu", 5: "bwd_ln_tanh", 6: "relu_mask", 7: "tg_bwd", 8: "dw"}
print("launches per update", per)
for i in used[-per:]:
    t = a[i]
    ok = t[:, 0] > 0
    t = t[ok]
    epi = int(t[0, 15] & 255); grid = int(t[0, 15] >> 8)
    nm = names[epi & 63] + ("_sk" if epi & 64 else "")
    t0 = t[:, 0].min()
    rel = lambda k: np.median((t[:, k] - t[:, 0]) / 1e3) if (t[:, k] > 0).all() else float("nan")
    span = (t[:, 4].max() - t0) / 1e3
    print(f"{i:3d} {nm:14s} grid {grid:4d} span {span:6.2f}  setup {rel(1):5.2f} wait {rel(2):5.2f} "
          f"xpre {rel(10):5.2f} prod_done {rel(11):5.2f} first {rel(8):5.2f} lastfull {rel(9):5.2f} mma_done {rel(3):5.2f} st5 {rel(5):5.2f} st13 {rel(13):5.2f} st14 {rel(14):5.2f} st6 {rel(6):5.2f} end {rel(4):5.2f} start_spread {(t[:,0].max()-t0)/1e3:5.2f}")
k = int(os.environ.get("TILES_OF", "-1"))
if k >= 0:
    i = used[-per:][k]
    t = a[i]; t0 = t[:, 0].min()
    for j in range(64):
        if t[j, 0] == 0: continue
        print(j, " ".join(f"{(t[j, s] - t0) / 1e3:6.2f}" if t[j, s] > 0 else "   -  " for s in (0, 2, 8, 9, 3, 5, 13, 14, 6, 7, 4)))
