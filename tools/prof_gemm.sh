#!/bin/bash
# Profiling variant of libjz with clock64 marks in the GEMM (per tile of CTA 0).
set -e
cd "$(dirname "$0")/.."
mkdir -p /tmp/jzprof
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DJZ_GEMM_PROF -Iinclude -c paper_2510_27002_b200/csrc/gemm.cu -o /tmp/jzprof/gemm.o
objs=""
for f in paper_2510_27002_b200/lib/obj/*.o; do b=$(basename $f); [ "$b" = gemm.o ] || objs="$objs $f"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o /tmp/jzprof/libjzg.so /tmp/jzprof/gemm.o $objs -Xcompiler -fPIC -lpthread -ldl -lrt
python - <<'PY'
import ctypes as C, torch, numpy as np, pathlib
import paper_2510_27002_b200._lib as L
L.LIB_PATH = pathlib.Path("/tmp/jzprof/libjzg.so")
L.ensure_device()
lib = L.load()
lib.jz_gemm_prof_read.argtypes = [C.c_void_p]
lib.jz_gemm_prof_dbg.argtypes = [C.c_int]
lib.jz_gemm_prof_ph.argtypes = [C.c_void_p]
import os
cases = [(148032, 1536, 512, 1, 0), (148032, 2048, 512, 3, 0), (148032, 2048, 512, 3, 4), (148032, 2048, 512, 3, 5), (148032, 2048, 512, 1, 0)]
for (M, N, K, epi, dbg) in cases:
    lib.jz_gemm_prof_dbg(dbg)
    A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(K, N, device="cuda").bfloat16()
    D = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
    aux = torch.zeros(M, N, device="cuda") if epi == 2 else None
    bias = torch.zeros(N, device="cuda")
    D2v = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for it in range(3):
        if it == 2: st.record()
        L.call("jz_gemm_bf16", A.data_ptr(), K, 1, B.data_ptr(), N, 0, D.data_ptr(), N, M, N, K, epi, bias.data_ptr(),
               None if aux is None else aux.data_ptr(), N, None if epi != 3 else D2v.data_ptr(), N, 1, None, L.stream_ptr())
    en.record(); torch.cuda.synchronize()
    us = st.elapsed_time(en) * 1e3
    D2 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if epi == 3 else None
    buf = np.zeros(64 * 8, dtype=np.uint64)
    lib.jz_gemm_prof_read(buf.ctypes.data)
    ph = np.zeros(64 * 4, dtype=np.int64)
    lib.jz_gemm_prof_ph(ph.ctypes.data)
    ph = ph.reshape(64, 4) // 3  # three launches accumulated
    t = buf.reshape(64, 8).astype(np.int64)
    print(f"M={M} N={N} K={K} epi={epi} dbg={dbg}: {us:.1f} us  {2*M*N*K/us/1e6:.0f} TF/s")
    base = t[2, 0]
    for ti in range(2, 6):
        r = t[ti] - base
        print(f"  tile {ti}: mma start {r[0]:7d} tempty ok {r[1]:7d} (+{t[ti,1]-t[ti,0]:5d}) mainloop issued {r[2]:7d} (+{t[ti,2]-t[ti,1]:5d}) | "
              f"epi wait {r[3]:7d} tfull {r[4]:7d} (+{t[ti,4]-t[ti,3]:5d}) epi done {r[5]:7d} (+{t[ti,5]-t[ti,4]:5d}) fullwait {t[ti,6]:5d} | phases wait/tmem/math/store {ph[ti].tolist()}")
PY
