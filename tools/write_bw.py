import torch
x = torch.empty(4 * 1024**3, dtype=torch.float32, device="cuda")  # 16 GiB
for name, fn in [("zero_", lambda: x.zero_()), ("fill_", lambda: x.fill_(1.5))]:
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ms = min(ts)
    print(f"{name}: {ms:.3f} ms  {x.numel()*4/ms/1e6:.0f} GB/s")
