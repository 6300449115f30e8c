"""Measure the dense int8 / bf16 / fp8 tensor-core peaks on this B200 with cuBLAS
(torch._int_mm, torch.matmul, torch._scaled_mm), the way MEASURED_PEAKS.json measured
bf16: 8192^3, best of 10 (burst) and a ~4 s back-to-back loop (sustained), CUDA events.
Writes one JSON object to stdout."""
import json
import time

import torch


def bench(fn, flops, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    burst = flops / (best / 1e3) / 1e12
    n = 0
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    s.record()
    while time.time() - t0 < 4.0:
        for _ in range(20):
            fn()
        n += 20
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    sustained = flops * n / (s.elapsed_time(e) / 1e3) / 1e12
    return burst, sustained


def main():
    N = 8192
    out = {"gpu": torch.cuda.get_device_name(0), "n": N, "how": "cuBLAS via torch, 8192^3, 2*N^3 ops, best of 10 "
                                                                 "(burst) / 4 s loop (sustained), CUDA events"}
    a8 = torch.randint(0, 2, (N, N), dtype=torch.int8, device="cuda")
    b8 = torch.randint(0, 2, (N, N), dtype=torch.int8, device="cuda").t().contiguous().t()
    out["int8_tops"], out["int8_tops_sustained"] = bench(lambda: torch._int_mm(a8, b8), 2 * N ** 3)
    ab = torch.randn(N, N, dtype=torch.bfloat16, device="cuda")
    bb = torch.randn(N, N, dtype=torch.bfloat16, device="cuda")
    out["bf16_tflops"], out["bf16_tflops_sustained"] = bench(lambda: ab @ bb, 2 * N ** 3)
    try:
        af = ab.to(torch.float8_e4m3fn)
        bf = bb.to(torch.float8_e4m3fn).t().contiguous().t()
        one = torch.ones((), device="cuda")
        out["fp8_tflops"], out["fp8_tflops_sustained"] = bench(
            lambda: torch._scaled_mm(af, bf, scale_a=one, scale_b=one, out_dtype=torch.bfloat16), 2 * N ** 3)
    except Exception as ex:  # noqa: BLE001
        out["fp8_error"] = str(ex)[:200]
    # mxfp4 (e2m1 operands, UE8M0 scales per 32 elements), as the fp4 all-pairs kernel uses
    try:
        rup = lambda x, m: (x + m - 1) // m * m
        a4 = torch.full((N, N // 2), 0x22, dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
        b4 = torch.full((N, N // 2), 0x22, dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2).t()
        sa = torch.full((rup(N, 128) * rup(N // 32, 4),), 127, dtype=torch.uint8, device="cuda").view(torch.float8_e8m0fnu)
        sb = torch.full((rup(N, 128) * rup(N // 32, 4),), 127, dtype=torch.uint8, device="cuda").view(torch.float8_e8m0fnu)
        fn = lambda: torch._scaled_mm(a4, b4, scale_a=sa, scale_b=sb, out_dtype=torch.bfloat16)
        r = fn()
        out["fp4_check"] = float(r[0, 0])            # 1.0 * 1.0 summed over K = N
        out["fp4_tflops"], out["fp4_tflops_sustained"] = bench(fn, 2 * N ** 3)
    except Exception as ex:  # noqa: BLE001
        out["fp4_error"] = str(ex)[:300]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
