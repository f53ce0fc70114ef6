#!/usr/bin/env python3
"""Our shared-memory r2c/c2r FFT engine vs cuFFT (comparator only, via torch.fft)
on the BASELINE plane sizes; prints one JSON line per size. Both sides time
batched transforms of device-resident FP32 planes with CUDA events."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1709_09479_b200 import dcsc  # noqa: E402


def cufft_ms(H, W, batch, iters=20):
    x = torch.rand(batch, H, W, device="cuda", dtype=torch.float32)
    s = torch.fft.rfft2(x)
    for _ in range(3):
        torch.fft.rfft2(x)
        torch.fft.irfft2(s, s=(H, W))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        torch.fft.rfft2(x)
    b.record()
    torch.cuda.synchronize()
    r2c = a.elapsed_time(b) / iters
    a.record()
    for _ in range(iters):
        torch.fft.irfft2(s, s=(H, W))
    b.record()
    torch.cuda.synchronize()
    return r2c, a.elapsed_time(b) / iters


for (H, W), batch in [((128, 128), 256 * 16), ((100, 100), 100 * 25), ((64, 64), 2048 * 8), ((256, 256), 512 * 4)]:
    ours = dcsc.fft_timing((H, W), 32, batch)
    ref = cufft_ms(H, W, batch)
    bytes_rt = batch * H * W * 4 + batch * H * (W // 2 + 1) * 8  # one read + one write
    print(json.dumps({"grid": [H, W], "batch": batch, "ours_r2c_ms": ours[0], "ours_c2r_ms": ours[1],
                      "cufft_r2c_ms": ref[0], "cufft_c2r_ms": ref[1],
                      "ours_r2c_GBps": bytes_rt / ours[0] / 1e6, "cufft_r2c_GBps": bytes_rt / ref[0] / 1e6}))
