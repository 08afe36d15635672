"""Measured dense tensor peaks on this B200 for the dense path's roofline denominators, the way
MEASURED_PEAKS.json measures bf16 (library GEMM, best of 10, CUDA events):
  - FP4 (e2m1 operands, block-scaled) via torch._scaled_mm: this torch exposes the 1x16 NVFP4
    form (e4m3 scales per 16 elements) of cuBLASLt's block-scaled FP4 GEMM, which runs on the same
    tcgen05 FP4 tensor pipe as the dense path's kind::mxf4 MMAs (ncu: utcomma fp4, 32768 ops/cycle/SM);
  - int8 -> int32 via torch._int_mm;
  - bf16 for reference.
Ops = 2 * M * N * K per GEMM.  Prints one JSON line per measurement."""
import json
import sys

import torch


def bench(fn, flops, iters=10):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return flops / (best * 1e-3) / 1e12, best


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    dev = torch.device("cuda")
    flops = 2.0 * n * n * n
    out = []
    a = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
    b = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
    t, ms = bench(lambda: a @ b, flops)
    out.append({"bench": "bf16_matmul", "n": n, "tflops": t, "ms": ms})
    ai = torch.randint(-2, 3, (n, n), device=dev, dtype=torch.int8)
    bi = torch.randint(-2, 3, (n, n), device=dev, dtype=torch.int8).t().contiguous().t()
    try:
        t, ms = bench(lambda: torch._int_mm(ai, bi), flops)
        out.append({"bench": "int8_int_mm", "n": n, "tops": t, "ms": ms})
    except Exception as e:
        out.append({"bench": "int8_int_mm", "error": str(e)[:200]})
    try:
        fp4 = torch.float4_e2m1fn_x2
        a4 = torch.randint(0, 256, (n, n // 2), device=dev, dtype=torch.uint8).view(fp4)
        b4 = torch.randint(0, 256, (n, n // 2), device=dev, dtype=torch.uint8).view(fp4)
        # block scales: one e4m3 (1.0) per 16 elements along K
        sa = torch.full((n * (n // 16),), 0x38, device=dev, dtype=torch.uint8).view(torch.float8_e4m3fn)
        sb = torch.full((n * (n // 16),), 0x38, device=dev, dtype=torch.uint8).view(torch.float8_e4m3fn)
        f = lambda: torch._scaled_mm(a4, b4.t(), sa, sb, out_dtype=torch.bfloat16)
        t, ms = bench(f, flops)
        out.append({"bench": "fp4_block_scaled_mm", "n": n, "tflops": t, "ms": ms})
    except Exception as e:
        out.append({"bench": "fp4_block_scaled_mm", "error": str(e)[:300]})
    for o in out:
        o["gpu"] = torch.cuda.get_device_name()
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    main()
