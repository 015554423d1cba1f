"""Cost of the NVML queries used by the bench clock sampler (while the GPU is busy)."""
import time, threading, torch, pynvml as nv
nv.nvmlInit(); h = nv.nvmlDeviceGetHandleByIndex(0)
a = torch.randn(4096, 4096, dtype=torch.complex128, device="cuda")
stop = False
def load():
    while not stop:
        b = a @ a
        torch.cuda.synchronize()
t = threading.Thread(target=load); t.start()
for name, fn in [("clock", lambda: nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                 ("power", lambda: nv.nvmlDeviceGetPowerUsage(h)),
                 ("reasons", lambda: nv.nvmlDeviceGetCurrentClocksEventReasons(h))]:
    ts = []
    for _ in range(20):
        t0 = time.perf_counter(); fn(); ts.append((time.perf_counter() - t0) * 1e3); time.sleep(0.05)
    print(name, "ms: median %.3f max %.3f" % (sorted(ts)[10], max(ts)))
stop = True; t.join()
