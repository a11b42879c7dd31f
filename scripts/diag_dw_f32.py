import torch
torch.manual_seed(0)
x = (torch.rand(32000, 700, device="cuda") < 0.05).float()
g = torch.randn(32000, 128, device="cuda")
ref = g.double().t() @ x.double()
def err(a):
    return float(((a.double() - ref).abs() / ref.abs().clamp(min=1)).max())
print("plain", err(g.t() @ x))
for S in (8, 32):
    print("bmm", S, err(torch.bmm(g.view(S, -1, 128).transpose(1, 2), x.view(S, -1, 700)).sum(0)))
print("tf32 flag", torch.backends.cuda.matmul.allow_tf32, torch.get_float32_matmul_precision())
