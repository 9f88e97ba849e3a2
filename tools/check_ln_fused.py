"""Quick GPU check of the LN-fused GEMMs vs the unfused kernels."""
import sys; sys.path.insert(0, "/root/repo")
import torch
from paper_2510_27002_b200 import kernels as K, _lib as L
L.ensure_device()
torch.manual_seed(0)
for M in (148032, 1000, 300):
    Kd = 512
    a = (torch.randn(M, Kd, device="cuda") * 0.5).bfloat16()
    w = (torch.randn(Kd, 512, device="cuda") * 0.05).bfloat16()
    b = torch.randn(512, device="cuda") * 0.1
    res = torch.randn(M, 512, device="cuda")
    g = 1 + 0.1 * torch.randn(512, device="cuda"); be = 0.1 * torch.randn(512, device="cuda")
    x1, xn, m, r = K.linear_fwd_ln(a, w, b, res, g, be)
    ref_x = K.linear_fwd(a, w, b, epilogue=L.EPI_RESID, aux=res)
    ref_xn, ref_m, ref_r = K.layernorm_fwd(ref_x, g, be)
    torch.cuda.synchronize()
    print("fwd M", M, "x", float((x1 - ref_x).abs().max()), "xn", float((xn.float() - ref_xn.float()).abs().max()),
          "mean", float((m - ref_m).abs().max()), "rstd rel", float(((r - ref_r) / ref_r).abs().max()))
    for skip in (257,):
        if M % skip: continue
        x1s, xns, ms, rs = K.linear_fwd_ln(a, w, b, res, g, be, skip_period=skip)
        ref_y, _, _ = K.layernorm_fwd(ref_x, g, be, skip_period=skip)
        print("  skip", skip, float((xns.float() - ref_y.float()).abs().max()))
    # backward
    Kb = 1536
    dy = (torch.randn(M, Kb, device="cuda") * 0.1).bfloat16()
    wq = (torch.randn(512, Kb, device="cuda") * 0.05).bfloat16()
    x = torch.randn(M, 512, device="cuda") * 2 + 0.3
    mean = x.mean(1); rstd = 1 / torch.sqrt(x.var(1, unbiased=False) + 1e-5)
    dres0 = torch.randn(M, 512, device="cuda")
    outs = []
    for fused in (True, False):
        dres = dres0.clone(); dres_b = torch.empty(M, 512, device="cuda", dtype=torch.bfloat16)
        dg = torch.empty(512, device="cuda"); db = torch.empty(512, device="cuda"); dz = torch.empty(512, device="cuda")
        if fused:
            K.linear_dx_ln(dy, wq, x=x, mean=mean, rstd=rstd, gamma=g, dres=dres, dres_bf16=dres_b, dgamma=dg, dbeta=db, dbias=dz)
        else:
            dt = K.linear_dx(dy, wq, epilogue=L.EPI_BF16)
            K.layernorm_bwd(x, mean, rstd, g, dt, dres, accumulate=True, dres_bf16=dres_b, dgamma=dg, dbeta=db, dbias=dz)
        outs.append((dres, dres_b, dg, db, dz))
    torch.cuda.synchronize()
    f, u = outs
    rel = lambda p, q: float((p.float() - q.float()).norm() / q.float().norm())
    print("bwd M", M, "dres", rel(f[0] - dres0, u[0] - dres0), "dres_b", rel(f[1], u[1]), "dg", rel(f[2], u[2]), "db", rel(f[3], u[3]), "dz", rel(f[4], u[4]))
# timing at M=148032
M = 148032
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / n * 1e3
for Kd in (512, 2048):
    a = (torch.randn(M, Kd, device="cuda") * 0.5).bfloat16(); w = (torch.randn(Kd, 512, device="cuda") * 0.05).bfloat16()
    b = torch.randn(512, device="cuda") * 0.1; res = torch.randn(M, 512, device="cuda"); g = torch.ones(512, device="cuda"); be = torch.zeros(512, device="cuda")
    tf = t(lambda: K.linear_fwd_ln(a, w, b, res, g, be))
    tu = t(lambda: K.layernorm_fwd(K.linear_fwd(a, w, b, epilogue=L.EPI_RESID, aux=res), g, be))
    tg = t(lambda: K.linear_fwd(a, w, b, epilogue=L.EPI_RESID, aux=res))
    print(f"fwd K={Kd}: fused {tf:.1f} us, unfused {tu:.1f} us (gemm alone {tg:.1f})")
for Kb in (512, 1536, 2048):
    dy = (torch.randn(M, Kb, device="cuda") * 0.1).bfloat16(); wq = (torch.randn(512, Kb, device="cuda") * 0.05).bfloat16()
    x = torch.randn(M, 512, device="cuda"); mean = x.mean(1); rstd = 1 / torch.sqrt(x.var(1, unbiased=False) + 1e-5)
    dres = torch.randn(M, 512, device="cuda"); dres_b = torch.empty(M, 512, device="cuda", dtype=torch.bfloat16)
    dg = torch.empty(512, device="cuda"); db = torch.empty(512, device="cuda"); dz = torch.empty(512, device="cuda"); g = torch.ones(512, device="cuda")
    tf = t(lambda: K.linear_dx_ln(dy, wq, x=x, mean=mean, rstd=rstd, gamma=g, dres=dres, dres_bf16=dres_b, dgamma=dg, dbeta=db, dbias=dz))
    def unf():
        dt = K.linear_dx(dy, wq, epilogue=L.EPI_BF16)
        K.layernorm_bwd(x, mean, rstd, g, dt, dres, accumulate=True, dres_bf16=dres_b, dgamma=dg, dbeta=db, dbias=dz)
    tu = t(unf)
    tg = t(lambda: K.linear_dx(dy, wq, epilogue=L.EPI_BF16))
    print(f"bwd K={Kb}: fused {tf:.1f} us, unfused {tu:.1f} us (gemm alone {tg:.1f})")
