"""Probe: cuBLASLt int8 GEMM throughput on B200 (torch._int_mm), for the Ozaki Gram plan."""
import torch, time
dev = "cuda"
for (m, n, k) in [(6016, 6016, 2048), (6016, 6016, 8192), (6016, 6016, 28672), (8192, 8192, 8192)]:
    a = torch.randint(-127, 128, (m, k), dtype=torch.int8, device=dev)
    b = torch.randint(-127, 128, (k, n), dtype=torch.int8, device=dev).t().contiguous().t()
    for _ in range(3):
        c = torch._int_mm(a, b)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 10
    for _ in range(reps):
        c = torch._int_mm(a, b)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"int8 {m}x{n}x{k}: {ms:.3f} ms  {2*m*n*k/ms/1e9:.1f} TOPS")
    a16 = torch.randn(m, k, dtype=torch.bfloat16, device=dev); b16 = torch.randn(k, n, dtype=torch.bfloat16, device=dev)
    for _ in range(3): c = a16 @ b16
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): c = a16 @ b16
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"bf16 {m}x{n}x{k}: {ms:.3f} ms  {2*m*n*k/ms/1e9:.1f} TFLOPS")
