import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2109_04804_b200 import configs, hbpdc, inputs
cfg = configs.CONFIGS["C3"]
torch.cuda.set_stream(torch.cuda.Stream())
ctx = hbpdc.context_for(cfg)
co = ctx.node_coords()
W0 = inputs.initial_state("C3", co, noise=cfg.noise)
W = torch.tensor(W0, device="cuda")
n = ctx.n
sig = ctx.rhs(W)
g = torch.Generator().manual_seed(1)
dW = torch.randn(n, generator=g, dtype=torch.float64).cuda()
dS = torch.randn(n, generator=g, dtype=torch.float64).cuda()
flush = torch.empty(64*1024*1024, dtype=torch.float64, device="cuda")
st = ctx.stream
for mode in ["fd", "exact"]:
    o1, o2 = ctx.jvp(1.0, 1.0, 0.0145, W, sig, dW, dS, mode=mode)
    torch.cuda.synchronize()
    print(mode, "norms", o1.norm().item(), o2.norm().item(), "nan?", torch.isnan(o1).any().item())
    ts = []
    for r in range(10):
        flush.fill_(r)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st); ctx.jvp(1.0, 1.0, 0.0145, W, sig, dW, dS, mode=mode, out1=o1, out2=o2); e1.record(st)
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(mode, "ms", np.median(ts), "GB/s alg", 48*n/(np.median(ts)/1e3)/1e9)
a1, a2 = ctx.jvp(1.0, 1.0, 0.0145, W, sig, dW, dS, mode="fd")
b1, b2 = ctx.jvp(1.0, 1.0, 0.0145, W, sig, dW, dS, mode="exact")
print("fd vs exact rel", ((a1-b1).norm()**2 + (a2-b2).norm()**2).sqrt().item() / (b1.norm()**2+b2.norm()**2).sqrt().item())
r1 = ctx.rhs(W); ts=[]
for r in range(10):
    flush.fill_(r)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st); ctx.rhs(W, out=r1); e1.record(st); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print("R1 ms", np.median(ts), "GB/s alg", 16*n/(np.median(ts)/1e3)/1e9)
