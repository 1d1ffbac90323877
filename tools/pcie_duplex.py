"""PCIe copy rates on this box: H2D alone, D2H alone, H2D + D2H concurrently (pinned host
memory, 2.45 GB = one config-4 vector each way; CUDA events, best of 3).  The floor of the e2e
fd_apply_host_batch step is the concurrent pair's time."""
import json, torch
n = 305895744
h_r = torch.empty(n, dtype=torch.float64).pin_memory()
h_z = torch.empty(n, dtype=torch.float64).pin_memory()
d_r = torch.empty(n, dtype=torch.float64, device="cuda")
d_z = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn):
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); 
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
        e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best
def h2d():
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1): d_r.copy_(h_r, non_blocking=True)
def d2h():
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2): h_z.copy_(d_z, non_blocking=True)
def both():
    h2d(); d2h()
out = {}
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timed(fn)
    out[name] = {"ms": round(ms, 2), "GB/s per direction": round(8 * n / ms / 1e6, 1)}
print(json.dumps(out))
