"""fp32 reduction-to-L2 throughput for a fused dQ (atomic accumulation of 128x128 tiles)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2506_19852_b200 as P
    lib = ctypes.CDLL(P.debug_library_path())
    out = torch.zeros(148, dtype=torch.int64, device="cuda")
    for blocks in (929, 24 * 929):  # one head of H33 (61 MB) / all 24 heads (1.46 GB)
        buf = torch.zeros(blocks * 128 * 128, dtype=torch.float32, device="cuda")
        for mode in (0, 1):
            tiles = 64
            assert lib.radial_cuda_debug_red_rate(mode, ctypes.c_void_p(buf.data_ptr()), blocks, tiles,
                                                  ctypes.c_void_p(out.data_ptr())) == 0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lib.radial_cuda_debug_red_rate(mode, ctypes.c_void_p(buf.data_ptr()), blocks, tiles,
                                           ctypes.c_void_p(out.data_ptr()))
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            byts = 148 * tiles * 128 * 128 * 4
            print(f"blocks={blocks:6d} mode={'v4' if mode else 'scalar'}: {byts / ms / 1e9:8.1f} GB/s of fp32 adds "
                  f"({ms:.3f} ms, {byts / 1e9:.2f} GB)")
        del buf


if __name__ == "__main__":
    main()
