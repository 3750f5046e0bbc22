import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2502_00356_b200 as bg
from paper_2502_00356_b200 import besselk as B
for n in (1_000_000, 4_000_000):
    rng = np.random.default_rng(1)
    x = 140 * (1 - rng.random(n)); nu = 20 * (1 - rng.random(n))
    def t(reps=15):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize(); a = time.perf_counter(); bg.bessel_k_batch(x, nu); torch.cuda.synchronize(); ts.append(time.perf_counter() - a)
        return 1e3 * float(np.median(ts[5:]))
    for mc in (1 << 18, 1 << 22, 1 << 18, 1 << 22):
        B._HOST_MIN_CHUNK = mc
        print(n, 'min chunk', mc, '%.2f ms' % t(), flush=True)
