import time, sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2109_04804_b200 import configs, hbpdc, inputs
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
pc = sys.argv[2] if len(sys.argv) > 2 else "bjext"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = configs.CONFIGS[name]
kw = {}
if len(sys.argv) > 4: kw['restart'] = int(sys.argv[4])
ctx = hbpdc.context_for(cfg, precond=pc, **kw)
co = ctx.node_coords()
W0 = inputs.initial_state(name, co, noise=cfg.noise)
dt = configs.cfl_dt(cfg, inputs.initial_state(name, co))
print(name, "dt", dt, "n", ctx.n, flush=True)
W = torch.tensor(W0, device="cuda")
ctx.profile(True)
for s in range(steps):
    t = time.time(); st = ctx.step(dt, W); torch.cuda.synchronize()
    print("step", s, f"{time.time()-t:.3f}s", st, flush=True)
names = ["gemv", "jvp", "resid", "dots", "axpy", "kapply", "build"]
torch.cuda.set_stream(torch.cuda.Stream())
for k in range(7):
    n, ms, by = ctx.profile_read(k)
    print(f"{names[k]:8s} launches {n:6d} total {ms:9.2f} ms avg {ms/max(n,1):.4f} ms  {by/max(ms,1e-9)/1e6:8.1f} GB/s")
print("mem GB", torch.cuda.max_memory_allocated()/1e9, torch.cuda.mem_get_info())
