"""cuBLAS (torch.matmul, bf16) reference times for the ResNet-50 GEMM shapes — a
calibration point for tc_gemm, not part of the product path."""
import torch
shapes = [(50176, 1024, 256), (50176, 256, 1024), (12544, 2048, 512), (12544, 512, 2048),
          (200704, 512, 128), (802816, 64, 256), (802816, 256, 64), (16384, 4096, 4096)]
for M, K, N in shapes:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        c = a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"cuBLAS M={M} K={K} N={N}: {ms*1e3:.1f} us {2*M*N*K/ms/1e9:.1f} TF/s "
          f"{2*(M*K+M*N+K*N)/ms/1e6:.0f} GB/s")
