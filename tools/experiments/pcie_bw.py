"""PCIe copy rates from / to pinned host memory: H2D alone, D2H alone, both at once
(separate streams), for an 8.8 MB buffer (the bench's e2e per-step traffic)."""
import json
import torch

n = 4_521_984 // 4
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name, fn in [("h2d", lambda: d_a.copy_(h_in, non_blocking=True)),
                 ("d2h", lambda: h_out.copy_(d_b, non_blocking=True))]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        fn()
    e1.record()
    e1.synchronize()
    res[name + "_GBs"] = 50 * n * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
s1.wait_event(e0)
s2.wait_event(e0)
for _ in range(50):
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
e1.record()
e1.synchronize()
res["both_each_GBs"] = 50 * n * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9
print(json.dumps(res))
