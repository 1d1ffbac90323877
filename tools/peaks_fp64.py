"""Measure the FP64 roofline denominators on the B200 box.

cuBLAS DGEMM 8192^3 via torch.matmul (burst = best of 10; sustained = 4 s loop),
plus the register-only DMMA / DFMA microbenchmarks of tools/fp64_peak.cu.
Prints one JSON object.
"""
import json
import subprocess
import time
import os

import torch


def dgemm(n=8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(10):
        e0.record(); torch.matmul(a, b, out=c); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    burst = 2 * n ** 3 / (best * 1e-3) / 1e12
    t0 = time.time(); cnt = 0
    e0.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b, out=c); cnt += 1
        if cnt % 8 == 0:
            torch.cuda.synchronize()
    e1.record(); e1.synchronize()
    sus = 2 * n ** 3 * cnt / (e0.elapsed_time(e1) * 1e-3) / 1e12
    return burst, sus


def main():
    here = os.path.dirname(os.path.abspath(__file__))
    out = {"gpu": torch.cuda.get_device_name(0)}
    b, s = dgemm()
    out["cublas_dgemm_tflops_burst"] = round(b, 2)
    out["cublas_dgemm_tflops_sustained"] = round(s, 2)
    res = subprocess.run([os.path.join(here, "fp64_peak")], capture_output=True, text=True)
    out["micro"] = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
