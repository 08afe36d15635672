"""Measure the dense int8 tensor peak on this B200 the way MEASURED_PEAKS.json
measured bf16: best of 10 8192^3 GEMMs timed with CUDA events (cuBLASLt via
torch._int_mm), plus the bf16 figure again for a same-run ratio. Output: JSON lines.
This is a measurement tool for the roofline denominator only; nothing on the
product path calls it."""
import json
import torch


def best_ms(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    n = 8192
    a8 = torch.randint(-1, 2, (n, n), dtype=torch.int8, device="cuda")
    b8 = torch.randint(-1, 2, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    ms = best_ms(lambda: torch._int_mm(a8, b8))
    print(json.dumps({"bench": "int8_gemm_cublaslt", "n": n, "ms": ms, "TOPS": 2 * n**3 / ms / 1e9}))
    ab = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    bb = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    ms = best_ms(lambda: ab @ bb)
    print(json.dumps({"bench": "bf16_gemm_cublas", "n": n, "ms": ms, "TFLOPS": 2 * n**3 / ms / 1e9}))
    x = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
    y = torch.empty_like(x)
    ms = best_ms(lambda: y.copy_(x))
    print(json.dumps({"bench": "hbm_copy", "GBps": 2 * x.numel() * 2 / ms / 1e6}))


if __name__ == "__main__":
    main()
