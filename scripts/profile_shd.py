"""Kernel-time breakdown of the SHD-shaped training step (torch.profiler,
CUPTI) -- which kernels the 3-layer step spends its time in (GPU only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2501_14490_b200.net import Adam, build_task_net

dev = torch.device("cuda")
T, B, IN, H = 250, 128, 700, 128
k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
net = build_task_net(channels=H, num_layers=3, order=k, classes=20, seed=0, in_features=IN, device=dev)
g = torch.Generator(device=dev).manual_seed(5)
x = (torch.rand((T, B, IN), generator=g, device=dev) < 0.05).to(torch.float32)
y = torch.randint(0, 20, (B,), generator=g, device=dev)
opt = Adam(net.parameters_list(), 1e-3)
for _ in range(3):
    net.train_step_grads_async(x, y); opt.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        net.train_step_grads_async(x, y); opt.step()
    torch.cuda.synchronize()
rows = sorted(prof.key_averages(), key=lambda e: -e.self_device_time_total)
tot = sum(e.self_device_time_total for e in rows)
print(f"per step: {tot / 5:.1f} us of kernels")
for e in rows[:30]:
    print(f"{e.self_device_time_total / 5:8.1f} us/step {e.count // 5:4d}x  {e.key[:150]}")
