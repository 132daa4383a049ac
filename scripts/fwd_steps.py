"""Forward kernel time per KV step (sparse H33 union steps and dense), for variant libraries:
    RADIAL_CUDA_LIB=variants/x/libradial_cuda.so python scripts/fwd_steps.py
Prints ms and SM clocks per chunk-step (clock sampled with NVML during the timed loop)."""
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import pynvml
    import torch
    import paper_2506_19852_b200 as P
    pynvml.nvmlInit()
    hdl = pynvml.nvmlDeviceGetHandleByIndex(0)
    cfg = sys.argv[1] if len(sys.argv) > 1 else "hunyuan33"
    f, s, H = {"hunyuan33": (33, 3600, 24), "hunyuan132": (132, 3600, 24), "wan21": (21, 3600, 40),
               "mochi28": (28, 1590, 24)}[cfg]
    d, B = 128, 128
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    host = lay.host()
    rp, ci = host.row_ptr.astype(np.int64), host.col_idx.astype(np.int64)
    R = host.grid_rows
    union = sum(len(np.union1d(ci[rp[2 * p]:rp[2 * p + 1]], ci[rp[2 * p + 1]:rp[2 * p + 2]] if 2 * p + 1 < R else []))
                for p in range((R + 1) // 2))
    res = {"lib": os.path.basename(os.path.dirname(P.library_path())), "config": cfg}
    for name, fn, steps, it in (("sparse", lambda: P.masked_attention(q, k, v, lay), union * H, 10),
                                ("dense", lambda: P.dense_attention(q, k, v), ((R + 1) // 2) * R * H, 4)):
        if name == "dense" and cfg == "hunyuan132":
            continue
        for _ in range(3):
            fn()
        clk = []
        stop = threading.Event()

        def sample():
            while not stop.is_set():
                clk.append(pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM))
                time.sleep(0.01)
        th = threading.Thread(target=sample)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        th.start()
        e0.record()
        for _ in range(it):
            fn()
        e1.record()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        ms = e0.elapsed_time(e1) / it
        mhz = float(np.median(clk)) if clk else float("nan")
        res[name] = {"ms": round(ms, 3), "mhz": mhz, "clk_per_step": round(ms * 1e-3 * mhz * 1e6 * 148 / steps, 1)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
