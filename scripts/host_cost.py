import ctypes, time, torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_2501_14490_b200 as P
from paper_2501_14490_b200 import _lib as L
dev = torch.device('cuda', 0)
T,B,C,k,d = 1024,64,512,4,1
x = torch.randn((T,B,C), device=dev); dy = torch.randn((T,B,C), device=dev)
cfg = P.NeuronConfig(channels=C, order=k, dilation=d, quantized=True)
layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(1), device=dev)
lib = L.lib(); desc = L.make_desc(x.shape, k, d, torch.float32, flags=L.PSN_QUANTIZED | L.PSN_USE_BATCH_STATS)
ws = L.workspace(desc, dev); out = torch.empty_like(x); dx = torch.empty_like(x)
fold = torch.empty((C, L.fold_stride(k)), dtype=torch.float64, device=dev)
g = torch.empty(C*k+2*C, dtype=torch.float64, device=dev)
sp = torch.cuda.current_stream().cuda_stream
W, gam, bet, rm, rv = layer.W.detach(), layer.gamma.detach(), layer.beta.detach(), layer.running_mean, layer.running_var
def fwd():
    L.check(lib.psn_forward_train(ctypes.byref(desc), x.data_ptr(), W.data_ptr(), gam.data_ptr(), bet.data_ptr(), rm.data_ptr(), rv.data_ptr(), out.data_ptr(), fold.data_ptr(), ws.data_ptr(), sp))
def bwd():
    L.check(lib.psn_backward(ctypes.byref(desc), x.data_ptr(), dy.data_ptr(), W.data_ptr(), gam.data_ptr(), fold.data_ptr(), dx.data_ptr(), g[:C*k].data_ptr(), g[C*k:C*k+C].data_ptr(), g[C*k+C:].data_ptr(), ws.data_ptr(), sp))
for _ in range(5): fwd(); bwd()
torch.cuda.synchronize()
# host cost per call: enqueue behind a long sleep kernel so the GPU never drains
torch.cuda._sleep(200_000_000)
t0 = time.perf_counter()
for _ in range(50): fwd()
t1 = time.perf_counter()
for _ in range(50): bwd()
t2 = time.perf_counter()
torch.cuda.synchronize()
print(f"host enqueue fwd {1e6*(t1-t0)/50:.1f} us/call, bwd {1e6*(t2-t1)/50:.1f} us/call")
# device time back-to-back vs isolated
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
torch.cuda._sleep(50_000_000)
ev[0].record()
for _ in range(20): fwd(); bwd()
ev[1].record(); torch.cuda.synchronize()
print(f"queued (host-hidden) step {ev[0].elapsed_time(ev[1])/20*1000:.1f} us")
ev[2].record()
for _ in range(20): fwd(); bwd()
ev[3].record(); torch.cuda.synchronize()
print(f"direct step {ev[2].elapsed_time(ev[3])/20*1000:.1f} us")
# isolated vs alternating launches (device time per call)
def timed(fn_list, reps=20):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps * len(fn_list))]
    k = 0
    for _ in range(reps):
        for fn in fn_list:
            evs[k][0].record(); fn(); evs[k][1].record(); k += 1
    torch.cuda.synchronize()
    ts = [a.elapsed_time(b) * 1000 for a, b in evs]
    return [sum(ts[i::len(fn_list)]) / reps for i in range(len(fn_list))]
print("fwd only   %.1f us" % timed([fwd])[0])
print("bwd only   %.1f us" % timed([bwd])[0])
f_, b_ = timed([fwd, bwd])
print("alternating fwd %.1f us, bwd %.1f us" % (f_, b_))
# cost of a small stream memset (what each streamed launch does first)
import ctypes as _ct
_cudart = _ct.CDLL("libcudart.so") if False else None
def ms_only():
    torch.cuda.current_stream().synchronize()
zb = 24576
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100):
    ws[:zb].zero_()
e1.record(); torch.cuda.synchronize()
print("24 KB fill kernel: %.2f us each (back to back)" % (e0.elapsed_time(e1) * 10))
e0.record()
for _ in range(20):
    ws[:zb].zero_(); fwd()
e1.record(); torch.cuda.synchronize()
print("fill + fwd: %.1f us" % (e0.elapsed_time(e1) * 50))
# CUDA graph replay of one fwd+bwd step (cooperative launches captured)
try:
    s2 = torch.cuda.Stream()
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        sp_saved = sp
    g_ = torch.cuda.CUDAGraph()
    # the ctypes calls take the stream handle explicitly: capture on the current stream
    with torch.cuda.graph(g_):
        sp = torch.cuda.current_stream().cuda_stream
        fwd(); bwd()
    sp = sp_saved
    torch.cuda.synchronize()
    for _ in range(3): g_.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): g_.replay()
    e1.record(); torch.cuda.synchronize()
    print("graph replay step: %.1f us" % (e0.elapsed_time(e1) * 50))
except Exception as ex:
    print("graph capture failed:", repr(ex)[:300])
