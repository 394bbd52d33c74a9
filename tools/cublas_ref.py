"""cuBLAS bf16 GEMM reference shapes (torch.matmul) for comparing tensor-pipe utilisation
with the expert GEMMs under ncu.  Dev tool."""
import sys
import torch

M, N, K = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (131072, 3072, 768)))
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    c = a @ b
e.record()
e.synchronize()
ms = s.elapsed_time(e) / 10
print(f"M={M} N={N} K={K}: {ms:.3f} ms, {2 * M * N * K / ms / 1e9:.0f} TFLOP/s")
