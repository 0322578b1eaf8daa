"""cuBLAS DGEMM reference peak (torch.matmul fp64), burst and sustained,
measured the way MEASURED_PEAKS.json measures bf16: 2*N^3 flops, CUDA events."""
import json
import time

import torch


def main():
    out = {}
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device="cuda")
        b = torch.randn(n, n, dtype=torch.float64, device="cuda")
        for _ in range(3):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[f"dgemm_{n}_burst_tflops"] = 2 * n**3 / best / 1e9
        # sustained: back to back for ~4 s
        t0 = time.time()
        cnt = 0
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        while time.time() - t0 < 4.0:
            torch.matmul(a, b)
            cnt += 1
            if cnt % 8 == 0:
                torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        out[f"dgemm_{n}_sustained_tflops"] = 2 * n**3 * cnt / e0.elapsed_time(e1) / 1e9
    # tall-skinny shapes of the path (cfg1): 20000x1000 @ 1000x60 and its transpose
    g = torch.randn(20000, 1000, dtype=torch.float64, device="cuda")
    x = torch.randn(1000, 60, dtype=torch.float64, device="cuda")
    q = torch.randn(20000, 60, dtype=torch.float64, device="cuda")
    for name, fn in (("gx", lambda: g @ x), ("gtq", lambda: g.t() @ q)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        out[f"cublas_{name}_cfg1_tflops"] = 2 * 20000 * 1000 * 60 / ms / 1e9
        out[f"cublas_{name}_cfg1_us"] = ms * 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
