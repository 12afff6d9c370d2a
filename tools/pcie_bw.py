"""Host link bandwidth on the GPU box: pinned H2D alone, D2H alone, and both directions at once on
two streams (the e2e path's ceiling; tools/, not a test)."""
import torch
n = 1 << 28  # 1 GiB of float32
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_in = torch.empty(n, dtype=torch.float32, device="cuda")
d_out = torch.zeros(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3
for _ in range(2):
    t_h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
    t_d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))
    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur); s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        cur.wait_stream(s1); cur.wait_stream(s2)
    t_both = timed(both)
gb = 4 * n / 1e9
print(f"H2D {gb / t_h2d:.1f} GB/s, D2H {gb / t_d2h:.1f} GB/s, both at once {2 * gb / t_both:.1f} GB/s aggregate "
      f"({t_both * 1e3:.1f} ms for {gb:.2f} GB each way)")
