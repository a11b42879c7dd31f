"""One traced fwd+bwd at the metric shape (PSN_TRACE=1): summarises the
per-CTA wait/compute breakdown the stream kernels print (bounded; GPU only)."""
import os, re, subprocess, sys

if os.environ.get("PSN_TRACE_CHILD"):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np, torch
    import paper_2501_14490_b200 as P
    T, B, C, k, d = (int(v) for v in sys.argv[1:6])
    cfg = P.NeuronConfig(channels=C, order=k, dilation=d, quantized=True)
    layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(1), device="cuda")
    x = torch.randn((T, B, C), device="cuda", requires_grad=True)
    dy = torch.randn((T, B, C), device="cuda")
    for _ in range(3):
        layer(x, P.Mode.TRAIN).backward(dy)
    torch.cuda.synchronize()
    os.environ["PSN_TRACE"] = "1"
    print("=== traced", flush=True)
    layer(x, P.Mode.TRAIN).backward(dy)
    torch.cuda.synchronize()
    sys.exit(0)

args = sys.argv[1:] or ["1024", "64", "512", "4", "1"]
env = dict(os.environ, PSN_TRACE_CHILD="1")
r = subprocess.run([sys.executable, __file__, *args], env=env, capture_output=True, text=True, timeout=300)
out = r.stdout.split("=== traced", 1)[-1]
open(os.environ.get("PSN_TRACE_RAW", "/dev/null"), "w").write(out)
rows = {}
for line in out.splitlines():
    m = re.match(r"PSNTRACE (\w+) (\w+) cta (\d+) (.*)", line)
    if not m:
        continue
    kv = dict(zip(m.group(4).split()[0::2], (int(v) for v in m.group(4).split()[1::2])))
    rows.setdefault((m.group(1), m.group(2)), []).append(kv)
for key, lst in sorted(rows.items()):
    keys = lst[0].keys()
    print(key, "n=%d" % len(lst))
    for kk in keys:
        vals = [r[kk] for r in lst]
        print("   %-9s mean %10.1f  min %10d  max %10d" % (kk, sum(vals) / len(vals), min(vals), max(vals)))
print(r.stderr[-2000:] if r.returncode else "")
