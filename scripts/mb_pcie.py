"""PCIe copy bandwidth on the GPU box: pinned H2D alone, D2H alone, both at once
(the e2e bench line moves 268 MB each way per step at the metric shape)."""
import torch

n = 134217728 // 4 * 2  # 268 MB of f32
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_in = torch.empty(n, dtype=torch.float32, device="cuda")
d_out = torch.zeros(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps):
        fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


gb = n * 4 / 1e9
for name, fn in (("H2D", h2d), ("D2H", d2h), ("both", both)):
    ms = timed(fn)
    print(f"{name:5s} {ms:7.2f} ms  {gb / ms * 1e3:6.1f} GB/s per direction")
