"""Time the 256 MiB L2 flush variants (uint8 / int32 / int64 fill) with CUDA events."""
import torch
buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
views = {"u8": buf, "i32": buf.view(torch.int32), "i64": buf.view(torch.int64)}
for name, v in views.items():
    for _ in range(3):
        v.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(20):
        v.fill_(k)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"{name}: {ms * 1e3:.1f} us per 256 MiB fill = {256 * 2**20 / ms / 1e9:.0f} GB/s")
