"""Prefill throughput with the SM clock sampled during the run (NVML): is the
config-3 number limited by the kernel or by the clock the GPU holds under the
tensor-core load? Runs the prefill back to back for ~3 s per shape and reports
TFLOP/s, the median SM clock, throttle reasons, and the tensor-pipe roofline at
that clock (148 SMs x 8192 dense bf16 FLOP/clk; M128xN128xK16 = 64.4 clk
measured with tools/mma_probe.cu)."""
import json
import sys
import time

import torch

sys.path[:0] = [".", "tools"]
import bench
import kernel_bench as kb


class A:
    pass


for B, prefix, n_new in ((16, 2048, 512), (16, 8192, 512), (4, 0, 4096)):
    args = A()
    args.pf_batch, args.pf_prefix, args.pf_new, args.iters, args.warmup = B, prefix, n_new, 20, 3
    r = kb.bench_prefill(args, {"bf16_tflops": 1, "bf16_tflops_sustained": 1})[0]
    reps = max(3, int(3.0 / (r["us"] * 1e-6 * 20)))
    args.iters = 20 * reps
    with bench.ClockSampler(0) as clk:
        r = kb.bench_prefill(args, {"bf16_tflops": 1, "bf16_tflops_sustained": 1})[0]
    c = clk.summary()
    peak_at_clock = 148 * 8192 * c["sm_mhz"] * 1e6 / 1e12 if c["sm_mhz"] else None
    print(json.dumps({"config": r["config"], "us": r["us"], "TFLOP/s": r["TFLOP/s"], "clocks": c,
                      "tensor_peak_at_clock_TFLOPs": round(peak_at_clock, 1) if peak_at_clock else None,
                      "frac_of_peak_at_clock": round(r["TFLOP/s"] / peak_at_clock, 4) if peak_at_clock else None}))
