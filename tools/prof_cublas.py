import torch, sys
M, N, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    c = a @ b.t()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    c = a @ b.t()
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"cublas {M}x{N}x{K}: {ms:.3f} ms {2*M*N*K/ms/1e9:.1f} TF/s")
