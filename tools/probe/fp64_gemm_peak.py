"""Measure cuBLAS FP64 DGEMM / ZGEMM throughput via torch (the FP64 roofline denominator).
Burst = best of 10; sustained = back-to-back for ~4 s. Prints JSON lines."""
import json, time, torch

def bench(dtype, n, reps=10, sustain_s=4.0):
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    b = torch.randn(n, n, dtype=dtype, device="cuda")
    c = torch.empty(n, n, dtype=dtype, device="cuda")
    flop = (8.0 if dtype.is_complex else 2.0) * n ** 3
    for _ in range(2):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); torch.matmul(a, b, out=c); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e))
    # sustained
    cnt = 0
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time(); s.record()
    while time.time() - t0 < sustain_s:
        for _ in range(4):
            torch.matmul(a, b, out=c); cnt += 1
        torch.cuda.synchronize()
    e.record(); e.synchronize()
    sus = s.elapsed_time(e) / cnt
    return {"dtype": str(dtype), "n": n, "burst_tflops": flop / best / 1e9, "sustained_tflops": flop / sus / 1e9}

if __name__ == "__main__":
    print(json.dumps({"device": torch.cuda.get_device_name(0)}))
    for dt, n in [(torch.float64, 8192), (torch.complex128, 4096), (torch.complex128, 8192)]:
        print(json.dumps(bench(dt, n)), flush=True)
