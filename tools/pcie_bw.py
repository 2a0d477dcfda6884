"""Pinned host <-> device copy bandwidth on this box (the e2e floor): the HV
call's inputs (2.19 GB H2D) and output (0.73 GB D2H), alone and overlapped."""
import torch
n_in, n_out = 2194145280 // 2, 731381760 // 2
h_in = torch.empty(n_in, dtype=torch.bfloat16).pin_memory()
h_out = torch.empty(n_out, dtype=torch.bfloat16).pin_memory()
d_in = torch.empty(n_in, dtype=torch.bfloat16, device="cuda")
d_out = torch.empty(n_out, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))
def both():
    ev = torch.cuda.Event(); ev.record()
    with torch.cuda.stream(s1):
        s1.wait_event(ev); d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        s2.wait_event(ev); h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
ov = timed(both)
print(f"H2D 2.19 GB: {h2d:.2f} ms ({2194145280 / h2d / 1e6:.1f} GB/s); D2H 0.73 GB: {d2h:.2f} ms "
      f"({731381760 / d2h / 1e6:.1f} GB/s); both overlapped: {ov:.2f} ms")
