"""Library fp4 GEMM peak on this GPU: torch._scaled_mm on float4_e2m1fn_x2
operands with block-16 e4m3 scales (cuBLASLt NVFP4), 8192^3 and 16384^3."""
import torch, time
dev = "cuda"
for n in (8192, 16384):
    try:
        a = torch.randint(0, 256, (n, n // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        b = torch.randint(0, 256, (n, n // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        # NVFP4: block-16 e4m3 scales (1.0 = 0x38); same tensor rate as MXFP4 (kind::mxf4nvf4)
        sa = torch.full((n * (n // 16),), 0x38, dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)
        sb = torch.full((n * (n // 16),), 0x38, dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)
        f = lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"fp4 scaled_mm {n}^3: {2 * n ** 3 / ms / 1e9:.1f} TFLOP/s ({ms:.3f} ms)")
    except Exception as ex:
        print("fp4 scaled_mm failed:", type(ex).__name__, str(ex)[:2000]); break
for n in (8192,):
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev).t()
    torch._int_mm(a, b); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): torch._int_mm(a, b)
    e1.record(); torch.cuda.synchronize()
    print(f"int8 _int_mm {n}^3: {2 * n ** 3 / (e0.elapsed_time(e1) / 20) / 1e9:.1f} TOP/s")
