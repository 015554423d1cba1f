"""One cuBLAS ZGEMM at a filter shape (for an ncu look at the library kernel)."""
import sys
import torch
n, w = int(sys.argv[1]), int(sys.argv[2])
h = torch.randn(n, n, dtype=torch.complex128, device="cuda")
y = torch.randn(n, w, dtype=torch.complex128, device="cuda")
for _ in range(3):
    z = h @ y
torch.cuda.synchronize()
print("ok")
