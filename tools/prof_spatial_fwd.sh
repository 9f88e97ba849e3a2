#!/bin/bash
# Build a clock64-timeline variant of the spatial forward into lib/dbgf and print CTA 0's unit timelines.
set -e
cd "$(dirname "$0")/.."
if [ "$1" != "--run" ]; then
  mkdir -p paper_2510_27002_b200/lib/dbgf
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -DJZ_SPATIAL_FWD_PROF $EXTRA -Iinclude \
    -c paper_2510_27002_b200/csrc/attn_spatial.cu -o paper_2510_27002_b200/lib/dbgf/attn_spatial.o
  objs=""
  for f in paper_2510_27002_b200/lib/obj/*.o; do b=$(basename $f); [ "$b" = attn_spatial.o ] || objs="$objs $f"; done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2510_27002_b200/lib/dbgf/libjz.so \
    paper_2510_27002_b200/lib/dbgf/attn_spatial.o $objs -Xcompiler -fPIC -lpthread -ldl -lrt
  exit 0
fi
python - <<'PY'
import ctypes as C, os, pathlib, numpy as np, torch
import paper_2510_27002_b200._lib as L
L.LIB_PATH = pathlib.Path("paper_2510_27002_b200/lib/dbgf/libjz.so").resolve()
from paper_2510_27002_b200 import kernels as Kn
L.ensure_device()
S = int(os.environ.get("S", "257"))
frames, H, D = 576, 8, 512
qkv = torch.randn(frames * S, 3 * D, device="cuda").bfloat16()
for _ in range(3):
    out, olo, lse = Kn.attn_spatial_fwd(qkv, frames, S, H, keep_lo=True)
torch.cuda.synchronize()
lib = L.load()
buf = np.zeros(16 * 64, dtype=np.uint64)
lib.jz_attn_fwd_prof_read.argtypes = [C.c_void_p]
assert lib.jz_attn_fwd_prof_read(buf.ctypes.data) == 0
t = buf.reshape(16, 64).astype(np.int64)
names = {0: "MMA qk_full", 1: "MMA S0 issue", 2: "MMA S1 issue", 3: "MMA v_full", 4: "MMA PV0 issue", 5: "MMA PV1 issue",
         30: "TMA qk load", 31: "TMA v load", 40: "TAIL wait k", 41: "TAIL k_full", 42: "TAIL q0_full", 43: "TAIL col done",
         44: "TAIL wait v", 45: "TAIL v_full", 46: "TAIL v done"}
for tt in range(2):
    names[8 + tt] = f"SMX{tt} wait s_full"; names[10 + tt] = f"SMX{tt} s_full"; names[12 + tt] = f"SMX{tt} exp turn"
    names[14 + tt] = f"SMX{tt} max done"; names[16 + tt] = f"SMX{tt} P done"; names[18 + tt] = f"SMX{tt} o_full"
    names[20 + tt] = f"SMX{tt} epi done"; names[22 + tt] = f"SMX{tt} O loaded"; names[24 + tt] = f"SMX{tt} staged"
    names[26 + tt] = f"SMX{tt} staged (all warps)"
for u in (3, 4):
    base = t[u, 0]
    print(f"unit {u}: period {t[u + 1, 0] - base} cycles (MMA qk_full to next unit's)")
    for k in sorted(names, key=lambda k: t[u, k]):
        if t[u, k]:
            print(f"   {names[k]:22s} {t[u, k] - base:8d}")
PY
