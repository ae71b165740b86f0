"""HBM calibration for the PW traffic shape: 3 reads + 3 writes per point.

    python tools/membench.py     (needs tools/libmembench.so: nvcc -shared tools/membench.cu)
"""
import ctypes
import json
import subprocess
from pathlib import Path

import torch

HERE = Path(__file__).resolve().parent
SO = HERE / "libmembench.so"


def build():
    subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                    "-Xcompiler", "-fPIC", "-o", str(SO), str(HERE / "membench.cu")], check=True)


def main():
    if not SO.exists():
        build()
    L = ctypes.CDLL(str(SO))
    L.mb_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                         ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    n = 514 * 514 * 64  # one C1 field
    ins = [torch.randn(n, dtype=torch.float64, device="cuda") for _ in range(3)]
    outs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3)]
    pin = (ctypes.c_void_p * 3)(*[t.data_ptr() for t in ins])
    pout = (ctypes.c_void_p * 3)(*[t.data_ptr() for t in outs])
    st = torch.cuda.current_stream().cuda_stream
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for which, name, nbytes in ((0, "copy3", 6 * 8 * n), (1, "copy1", 2 * 8 * n), (2, "read3", 3 * 8 * n),
                                (3, "write3", 3 * 8 * n)):
        for grid_mult, block in ((4, 256), (8, 256), (16, 256), (32, 256), (4, 1024)):
            g = sms * grid_mult
            f = lambda: L.mb_run(which, pin, pout, n // 2, g, block, ctypes.c_void_p(st))  # noqa: E731
            for _ in range(5):
                f()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(50):
                f()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 50
            print(json.dumps({"kernel": name, "grid": g, "block": block, "ms": round(ms, 4),
                              "GBs": round(nbytes / (ms / 1e3) / 1e9, 1)}))
    # staging paths (one CTA per SM, contiguous region per CTA)
    L.mb_stage.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                           ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    big = torch.empty(3 * n, dtype=torch.float64, device="cuda").normal_()
    sink = torch.zeros(4, dtype=torch.float64, device="cuda")
    for mode, mname in ((0, "bulk"), (1, "cp.async"), (2, "ldg+sts")):
        for chunk, stages, ctas_per_sm, block in ((7168, 8, 1, 384), (7168, 16, 1, 384), (21504, 8, 1, 384),
                                                  (2048, 32, 1, 384), (4096, 32, 1, 384),
                                                  (16384, 12, 1, 384), (7168, 8, 2, 192), (7168, 4, 4, 128)):
            g = sms * ctas_per_sm
            per_cta = (3 * n * 8 // g) // chunk * chunk
            if stages * chunk > 220 * 1024 // ctas_per_sm:
                continue
            f = lambda: L.mb_stage(ctypes.c_void_p(big.data_ptr()), per_cta, chunk, stages, mode, g, block,  # noqa: E731
                                   ctypes.c_void_p(sink.data_ptr()), ctypes.c_void_p(st))
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                f()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 20
            print(json.dumps({"stage": mname, "chunk": chunk, "stages": stages, "ctas_per_sm": ctas_per_sm,
                              "ms": round(ms, 4), "read_GBs": round(per_cta * g / (ms / 1e3) / 1e9, 1)}))
    # torch references
    for label, fn, nb in (("torch_copy3", lambda: [o.copy_(i) for o, i in zip(outs, ins)], 6 * 8 * n),
                          ("torch_copy1", lambda: outs[0].copy_(ins[0]), 2 * 8 * n)):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 50
        print(json.dumps({"kernel": label, "ms": round(ms, 4), "GBs": round(nb / (ms / 1e3) / 1e9, 1)}))


if __name__ == "__main__":
    main()
