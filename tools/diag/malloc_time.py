import torch, time
x = []
t = []
for i in range(20):
    t0 = time.perf_counter(); y = torch.empty(6_553_600 // 16 * 16, dtype=torch.uint8, device="cuda"); torch.cuda.synchronize(); t.append(time.perf_counter() - t0); x.append(y)
print("cudaMalloc 6.5MB ms:", [round(v * 1e3, 2) for v in t])
