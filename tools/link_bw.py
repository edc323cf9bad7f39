"""Host-link bandwidth probe: one 4 GiB pinned D2H and H2D copy (the e2e bound of bench.py)."""
import time, torch
x = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
y = torch.empty(4 << 30, dtype=torch.uint8, pin_memory=True)
for direction in ("d2h", "h2d"):
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        if direction == "d2h": y.copy_(x, non_blocking=True)
        else: x.copy_(y, non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(direction, round(x.numel() / dt / 1e9, 1), "GB/s")
