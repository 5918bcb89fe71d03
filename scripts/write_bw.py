"""Write-only HBM bandwidth ceilings on this GPU (context for the fill roofline)."""
import json
import torch

torch.cuda.init()
res = {}
nbytes = 470 * 2**20
for name, dtype in (("u8", torch.uint8), ("f32", torch.float32)):
    x = torch.empty(nbytes // torch.tensor([], dtype=dtype).element_size(), dtype=dtype, device="cuda")
    for _ in range(3):
        x.fill_(1)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(10):
        s.record(); x.fill_(2); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    res[f"fill_{name}_GBps"] = nbytes / (best / 1e3) / 1e9
    best = 1e9
    for _ in range(10):
        s.record(); x.zero_(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    res[f"zero_{name}_GBps"] = nbytes / (best / 1e3) / 1e9
a = torch.empty(nbytes // 2, dtype=torch.uint8, device="cuda")
b = torch.empty_like(a)
for _ in range(3):
    b.copy_(a)
best = 1e9
for _ in range(10):
    s.record(); b.copy_(a); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
res["copy_rw_GBps"] = 2 * a.numel() / (best / 1e3) / 1e9
print(json.dumps(res))
