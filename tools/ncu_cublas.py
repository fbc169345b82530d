"""One cuBLAS DGEMM (measurement reference only; never on the product path)."""
import torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
c = a @ b; torch.cuda.synchronize()
c = a @ b; torch.cuda.synchronize()
