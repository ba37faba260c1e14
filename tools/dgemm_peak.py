"""cuBLAS DGEMM cross-check of the FP64 peak ('cuBLAS DGEMM 8192^3
as a cross-check only'). Prints one JSON line. Library code; not part of the product path."""
import json
import torch

def main():
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5):
        e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"dgemm_n": n, "dgemm_ms": best, "dgemm_tflops": 2 * n**3 / (best * 1e-3) / 1e12}))

if __name__ == "__main__":
    main()
