"""cuBLAS DGEMM 8192^3 throughput (FP64 library reference for SURVEY.md §8d), with clocks.

Library call on purpose: this is the FP64 denominator probe, not product code.
"""
import json, subprocess, time
import torch

def main():
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    # sustained: back to back for ~3 s while sampling clocks
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, text=True)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    k = 0; e0.record(); t = time.time()
    while time.time() - t < 3.0:
        torch.matmul(a, b); k += 1
        if k % 4 == 0: torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    smi.terminate(); out = smi.communicate()[0].strip().splitlines()
    ms = e0.elapsed_time(e1) / k
    clocks = sorted(int(float(l.split(",")[0])) for l in out if l.strip())
    print(json.dumps({"probe": "cublas_dgemm_8192", "burst_tflops": 2 * n**3 / best / 1e9,
                      "sustained_tflops": 2 * n**3 / ms / 1e9,
                      "sm_mhz_median": clocks[len(clocks) // 2] if clocks else None,
                      "smi_tail": out[-3:]}))

if __name__ == "__main__":
    main()
