"""Probe: PCIe H2D / D2H / duplex and device-copy bandwidth at the bench's
sizes (context for the e2e leg and the HBM roofline; not a bench number)."""
import json

import torch


def timed(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


n = 256 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
out = {}
out["h2d_GBs"] = n / timed(lambda: d_a.copy_(h_in, non_blocking=True)) / 1e6
out["d2h_GBs"] = n / timed(lambda: h_out.copy_(d_b, non_blocking=True)) / 1e6


def duplex():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t = timed(duplex)
out["duplex_ms_256MiB_each_way"] = t
out["duplex_total_GBs"] = 2 * n / t / 1e6
for mib in (256, 512, 2048):
    m = mib << 20
    a = torch.empty(m, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    out[f"d2d_copy_{mib}MiB_GBs_rw"] = 2 * m / timed(lambda: b.copy_(a)) / 1e6
print(json.dumps(out))
