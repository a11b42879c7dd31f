import time, pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
for f, name in ((lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), "clock"), (lambda: pynvml.nvmlDeviceGetCurrentClocksEventReasons(h), "reasons")):
    t = time.perf_counter()
    for _ in range(20): f()
    print(name, (time.perf_counter() - t) / 20 * 1e3, "ms")
