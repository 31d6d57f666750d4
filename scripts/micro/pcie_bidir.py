"""Dev microbenchmark: host link bandwidth H2D, D2H, and both at once
(pinned memory, separate streams), and in 7 / 6 array pieces."""
import time, torch
n = 1 << 28  # 1 GiB of f32
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True).fill_(1)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_in = torch.empty(n, dtype=torch.float32, device="cuda")
d_out = torch.empty(n, dtype=torch.float32, device="cuda").fill_(2)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=5):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    return reps * 4 * n / dt / 1e9
print(f"h2d {run(True, False):.1f} GB/s  d2h {run(False, True):.1f} GB/s  both(each) {run(True, True):.1f} GB/s")
