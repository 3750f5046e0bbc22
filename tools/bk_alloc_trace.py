import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2502_00356_b200 as bg
n = 64 << 20
rng = np.random.default_rng(20250201)
x = 140.0 * (1.0 - rng.random(n)); nu = 20.0 * (1.0 - rng.random(n))
for i in range(12):
    st0 = torch.cuda.host_memory_stats()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    bg.bessel_k_batch(x, nu)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    st1 = torch.cuda.host_memory_stats()
    print(i, round(dt * 1e3, 1), "host allocs", st1.get("num_host_alloc", 0) - st0.get("num_host_alloc", 0),
          "alloc MB", (st1.get("allocation.current", 0)), flush=True)
