#!/bin/bash
# Build a profiling variant of libjz (clock64 marks in the spatial backward) into /tmp and run it.
set -e
cd "$(dirname "$0")/.."
mkdir -p /tmp/jzprof
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DJZ_ATTN_PROF -Iinclude -c paper_2510_27002_b200/csrc/attn_spatial.cu -o /tmp/jzprof/attn_spatial.o
objs=""
for f in paper_2510_27002_b200/lib/obj/*.o; do b=$(basename $f); [ "$b" = attn_spatial.o ] || objs="$objs $f"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o /tmp/jzprof/libjz.so /tmp/jzprof/attn_spatial.o $objs -Xcompiler -fPIC -lpthread -ldl -lrt
python - <<'PY'
import ctypes as C, torch, numpy as np
import paper_2510_27002_b200._lib as L
L.LIB_PATH = __import__("pathlib").Path("/tmp/jzprof/libjz.so")
L.ensure_device()
lib = L.load()
import os
frames, S, H = 576, int(os.environ.get("S", "257")), 8
D = H * 64
qkv = torch.randn(frames * S, 3 * D, device="cuda").bfloat16()
out = torch.empty(frames * S, D, device="cuda", dtype=torch.bfloat16)
olo = torch.empty(frames * S, D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(frames, H, S, device="cuda")
dq = torch.empty_like(qkv)
WS = torch.empty(frames * H * 780, device='cuda')
L.call("jz_attn_spatial_fwd", qkv.data_ptr(), frames, S, H, 64, out.data_ptr(), olo.data_ptr(), lse.data_ptr(), L.stream_ptr())
for _ in range(3):
    L.call("jz_attn_spatial_bwd", qkv.data_ptr(), out.data_ptr(), olo.data_ptr(), out.data_ptr(), lse.data_ptr(), frames, S, H, 64, dq.data_ptr(), WS.data_ptr(), None, L.stream_ptr())
torch.cuda.synchronize()
buf = np.zeros(64 * 32, dtype=np.uint64)
lib.jz_attn_prof_read.argtypes = [C.c_void_p]
assert lib.jz_attn_prof_read(buf.ctypes.data) == 0
t = buf.reshape(32, 64).astype(np.int64)
names = {0: "MMA start", 1: "MMA load_full", 26: "EW prep_ready", 43: "HLP prep+load", 45: "HLP tail done", 46: "HLP dkdv_full0",
         47: "HLP epi0 done", 48: "HLP prepare done", 49: "HLP dkdv_full1", 50: "HLP epi1 done", 51: "HLP dq_full", 52: "HLP dq done",
         53: "TMA issue"}
for x in range(8):
    names[2 + x] = f"MMA sdp issued {x}"; names[10 + x] = f"MMA pds_full {x}"; names[18 + x] = f"MMA grad issued {x}"
    names[27 + x] = f"EW sdp_full {x}"; names[35 + x] = f"EW pds done {x}"
for u in (2, 3, 10):
    base = t[u, 0]
    print(f"unit {u}: total {t[u + 1, 0] - base} cycles")
    for k in sorted(names, key=lambda k: t[u, k]):
        if t[u, k]:
            print(f"   {names[k]:20s} {t[u, k] - base:8d}")
PY
