"""Timeline of the host-array BesselK pipeline (a traced replica of
besselk._bessel_k_host_pipelined): host stamps per phase and CUDA-event times."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_00356_b200 as bg  # noqa: E402
from paper_2502_00356_b200 import besselk as B, _lib  # noqa: E402

n = 64 << 20
rng = np.random.default_rng(20250201)
xf = 140.0 * (1.0 - rng.random(n))
nf = 20.0 * (1.0 - rng.random(n))
for _ in range(2):
    bg.bessel_k_batch(xf, nf, validate=False)
torch.cuda.synchronize()
dev = torch.device("cuda", 0)
cfg = bg.DEFAULT_CONFIG
T0 = time.perf_counter()
st = lambda: round((time.perf_counter() - T0) * 1e3, 2)
log = []
out_l = torch.empty(n, dtype=torch.float64, pin_memory=True)
out_k = torch.empty(n, dtype=torch.float64, pin_memory=True)
out_p = torch.empty(n, dtype=torch.uint8, pin_memory=True)
log.append(("alloc", st()))
comp = torch.cuda.current_stream(dev)
inp = torch.cuda.Stream(dev)
copy = torch.cuda.Stream(dev)
slots = B._stage_slots(torch, dev)
staged = [None, None]
freed = [None, None]
evs = []
e_start = torch.cuda.Event(enable_timing=True)
e_start.record(comp)
for ci, c0 in enumerate(range(0, n, B._HOST_CHUNK)):
    c1 = min(n, c0 + B._HOST_CHUNK)
    s = ci % 2
    if staged[s] is not None:
        staged[s].synchronize()
    a = st()
    sx, sn = slots[s]
    B._par_copy(sx.numpy()[:c1 - c0], xf[c0:c1])
    B._par_copy(sn.numpy()[:c1 - c0], nf[c0:c1])
    b = st()
    with torch.cuda.stream(inp):
        if freed[s] is not None:
            inp.wait_event(freed[s])
        h0 = torch.cuda.Event(enable_timing=True); h0.record(inp)
        xd = sx[:c1 - c0].to(dev, non_blocking=True)
        nd = sn[:c1 - c0].to(dev, non_blocking=True)
        ev_in = torch.cuda.Event(enable_timing=True)
        ev_in.record(inp)
    staged[s] = ev_in
    comp.wait_event(ev_in)
    xd.record_stream(comp)
    nd.record_stream(comp)
    logk, k, path = B._launch_besselk(xd, nd, cfg, _lib.ROUTE_HYBRID)
    done = torch.cuda.Event(enable_timing=True)
    done.record(comp)
    copy.wait_event(done)
    with torch.cuda.stream(copy):
        out_l[c0:c1].copy_(logk, non_blocking=True)
        out_k[c0:c1].copy_(k, non_blocking=True)
        out_p[c0:c1].copy_(path, non_blocking=True)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(copy)
    logk.record_stream(copy)
    k.record_stream(copy)
    path.record_stream(copy)
    freed[s] = ev
    evs.append((h0, ev_in, done, ev))
    log.append((f"chunk{ci} wait->{a} staged->{b} issued", st()))
copy.synchronize()
log.append(("end", st()))
for l in log:
    print(l)
for ci, (h0, hi, dn, dd) in enumerate(evs):
    print(ci, "H2D", round(e_start.elapsed_time(h0), 2), round(e_start.elapsed_time(hi), 2),
          "K end", round(e_start.elapsed_time(dn), 2), "D2H end", round(e_start.elapsed_time(dd), 2))
