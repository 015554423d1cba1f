import sys, time, torch, numpy as np
sys.path.insert(0, "/root/repo")
import paper_1206_3768_b200 as pkg
for n, nev in ((2048, 128), (5000, 500), (12000, 1200)):
    g = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    b = torch.eye(n, dtype=torch.complex128, device="cuda") + g @ g.conj().T / (4 * n)
    del g
    l = torch.linalg.cholesky(b).t().contiguous().t()
    y = torch.randn(n, nev, dtype=torch.complex128, device="cuda").t().contiguous().t()
    sol = pkg.EigenSolution(values=np.zeros(nev), vectors=y)
    pkg.back_transform(l, sol)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        pkg.back_transform(l, sol)
    torch.cuda.synchronize()
    print(f"back n={n} nev={nev}: {(time.perf_counter() - t) / 5 * 1e3:.2f} ms")
