#!/bin/bash
# Build a clock64-timeline variant of the v3 spatial backward into lib/dbg and print CTA 0's unit timelines.
set -e
cd "$(dirname "$0")/.."
if [ "$1" != "--run" ]; then
  mkdir -p paper_2510_27002_b200/lib/dbg
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -DJZ_SPATIAL_BWD_PROF $EXTRA -Iinclude \
    -c paper_2510_27002_b200/csrc/attn_spatial_bwd.cu -o paper_2510_27002_b200/lib/dbg/attn_spatial_bwd.o
  objs=""
  for f in paper_2510_27002_b200/lib/obj/*.o; do b=$(basename $f); [ "$b" = attn_spatial_bwd.o ] || objs="$objs $f"; done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2510_27002_b200/lib/dbg/libjz.so \
    paper_2510_27002_b200/lib/dbg/attn_spatial_bwd.o $objs -Xcompiler -fPIC -lpthread -ldl -lrt
  exit 0
fi
python - <<'PY'
import ctypes as C, os, pathlib, numpy as np, torch
import paper_2510_27002_b200._lib as L
L.LIB_PATH = pathlib.Path("paper_2510_27002_b200/lib/dbg/libjz.so").resolve()
from paper_2510_27002_b200 import kernels as Kn
L.ensure_device()
S = int(os.environ.get("S", "257"))
frames, H, D = 576, 8, 512
qkv = torch.randn(frames * S, 3 * D, device="cuda").bfloat16()
out, olo, lse = Kn.attn_spatial_fwd(qkv, frames, S, H, keep_lo=True)
dO = torch.randn(frames * S, D, device="cuda").bfloat16()
dq = torch.empty_like(qkv); cs = torch.empty(3 * D, device="cuda")
for _ in range(3):
    Kn.attn_spatial_bwd(qkv, out, dO, lse, frames, S, H, dqkv=dq, colsum=cs, out_lo=olo)
torch.cuda.synchronize()
lib = L.load()
buf = np.zeros(16 * 128, dtype=np.uint64)
lib.jz_attn_bwd3_prof_read.argtypes = [C.c_void_p]
assert lib.jz_attn_bwd3_prof_read(buf.ctypes.data) == 0
t = buf.reshape(16, 128).astype(np.int64)
names = {0: "TMA free_a", 1: "TMA free_b", 2: "TMA free_cd", 53: "HLP full_a", 54: "HLP ct done", 55: "HLP dkdv0 ready",
         56: "HLP epi0 done", 57: "HLP dq0 ready", 58: "HLP dq0 done", 59: "HLP dkdv1 ready", 60: "HLP epi1 done",
         61: "HLP dq1 ready", 62: "HLP dq1 done", 63: "HLP end"}
for x in range(10):
    names[3 + x] = f"MMA blk {x} S issue"; names[13 + x] = f"MMA blk {x} dP issue"; names[23 + x] = f"MMA grad {x}"
    names[33 + x] = f"PDS blk {x} start"; names[43 + x] = f"PDS blk {x} done"
    names[64 + x] = f"PDS blk {x} loaded"; names[74 + x] = f"PDS blk {x} computed"; names[84 + x] = f"PDS blk {x} st waited"
    names[94 + x] = f"PDS blk {x} proxy fenced"
tw = np.zeros(4 * 10 * 2 * 32, dtype=np.uint64)
lib.jz_attn_bwd3_tw_read.argtypes = [C.c_void_p]
assert lib.jz_attn_bwd3_tw_read(tw.ctypes.data) == 0
tw = tw.reshape(4, 10, 2, 32).astype(np.int64)
base = t[3, 3]
for x in range(10):
    ld = tw[3, x, 0, 2:18]; dn = tw[3, x, 1, 2:18]
    if ld.min() > 0:
        print(f"blk {x}: P/dS warps loaded {ld.min() - base}..{ld.max() - base}  done {dn.min() - base}..{dn.max() - base}  (warp order of done: {list(np.argsort(dn) + 2)})")
for u in (3,):
    base = t[u, 3]
    print(f"unit {u}: period {t[u + 1, 3] - base} cycles (MMA block-0 issue to next unit's)")
    for k in sorted(names, key=lambda k: t[u, k]):
        if t[u, k]:
            print(f"   {names[k]:22s} {t[u, k] - base:8d}")
PY
