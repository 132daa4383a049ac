"""tcgen05.mma issue/execute rate microbenchmark (clk per 128xNx16 MMA)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2506_19852_b200 as P
    lib = ctypes.CDLL(P.debug_library_path())
    names = {0: "SS N=128", 1: "TS N=128", 2: "SS N=256", 3: "TS N=256"}
    for ctas in (148,):
        for mode in [0, 1, 2, 3, 4, 5, 6, 7, 8, 9]:
            out = torch.zeros(ctas, dtype=torch.int64, device="cuda")
            iters = 2000
            assert lib.radial_cuda_debug_mma_rate(mode, iters, ctas, ctypes.c_void_p(out.data_ptr())) == 0
            cyc = out.double().mean().item() / (iters * 8)
            N = 64 if mode >= 6 else (256 if (mode & 2) else 128)
            print(f"ctas={ctas:4d} {names[mode & 3] if mode < 6 else ('SS N=64', 'TS N=64')[mode & 1]} nacc={(1 + ((mode >> 2) & 1)) if mode < 6 else (2 if mode < 8 else 1)}: {cyc:7.1f} clk/MMA  -> {128*N*16/cyc:7.0f} MAC/clk/SM")

    out = torch.zeros(149, dtype=torch.int64, device="cuda")
    for mode, nm in enumerate(["alone", "+tcgen05.ld (8 warps)", "+tcgen05.ld/st (8 warps)", "+ld.shared (8 warps)"]):
        iters = 2000
        assert lib.radial_cuda_debug_mma_interference(mode, iters, ctypes.c_void_p(out.data_ptr())) == 0
        cyc = out[:148].double().mean().item() / (iters * 8)
        print(f"SS N=128 MMA {nm:26s}: {cyc:6.1f} clk/MMA")


if __name__ == "__main__":
    main()
