"""Time the API-path transform / convolution kernels (config 1 shape and a large
batch) on device-resident int64 buffers through the C ABI; one JSON line.

    FNTGPU_LIB=build/ab/libfntgpu_X.so python tools/c1_probe.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_04253_b200 as P  # noqa: E402
from paper_2405_04253_b200 import _lib  # noqa: E402


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    lib = _lib.load()
    plan = P.default_plans()["cdc64"]
    dp = plan.device_plan()
    st = _lib.stream_handle()
    out = {}
    for batch in (16384, 1 << 20):
        g = torch.Generator(device="cuda").manual_seed(0)
        x = torch.randint(-16, 16, (batch, 64), device="cuda", dtype=torch.int64, generator=g)
        hb = torch.randint(-32, 32, (batch, 64), device="cuda", dtype=torch.int64, generator=g)
        h1 = hb[0].contiguous()
        z = torch.empty_like(x)
        y = torch.empty_like(x)
        conv_b = lambda: lib.fntgpu_cyclic_convolve_real(dp.handle, x.data_ptr(), hb.data_ptr(), 64,
                                                         z.data_ptr(), batch, 0, st)
        conv_1 = lambda: lib.fntgpu_cyclic_convolve_real(dp.handle, x.data_ptr(), h1.data_ptr(), 0,
                                                         z.data_ptr(), batch, 0, st)
        fwd = lambda: lib.fntgpu_fnt(dp.handle, 0, x.data_ptr(), y.data_ptr(), batch, 0, st)
        xi = torch.randint(-16, 16, (batch, 64), device="cuda", dtype=torch.int64, generator=g)
        hi = torch.randint(-32, 32, (batch, 64), device="cuda", dtype=torch.int64, generator=g)
        zi = torch.empty_like(x)
        cplx = lambda: lib.fntgpu_cyclic_convolve_complex(dp.handle, x.data_ptr(), xi.data_ptr(),
                                                          hb.data_ptr(), hi.data_ptr(), 64,
                                                          z.data_ptr(), zi.data_ptr(), batch, 0, st)
        for name, fn, words in (("conv_batched_h", conv_b, 3), ("conv_shared_h", conv_1, 2),
                                ("fnt", fwd, 2), ("conv_complex", cplx, 6)):
            us = timed(fn)
            out[f"{name}_{batch}"] = {"us": round(us, 2), "gelem_s": round(batch * 64 / us / 1e3, 1),
                                      "gbs": round(batch * 64 * 8 * words / us / 1e3, 1)}
        # parity spot check against the numpy restatement of the definition
        conv_b()
        torch.cuda.synchronize()
        xs, hs, zs = (t[:64].cpu().numpy() for t in (x, hb, z))
        F = 65537
        ref = np.zeros_like(xs)
        for k in range(64):
            ref = (ref + xs[:, k:k + 1] * np.roll(hs, k, axis=1)) % F
        out[f"parity_{batch}"] = bool((ref == zs % F).all())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
