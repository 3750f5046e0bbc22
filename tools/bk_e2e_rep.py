import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2502_00356_b200 as bg
n = 64 << 20
rng = np.random.default_rng(20250201)
x = 140.0 * (1.0 - rng.random(n)); nu = 20.0 * (1.0 - rng.random(n))
for v in (True, False, True, False):
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        bg.bessel_k_batch(x, nu, validate=v)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print("validate", v, [round(t * 1e3, 1) for t in ts])
