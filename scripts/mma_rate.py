"""tcgen05.mma issue/execute rate microbenchmark (clk per 128xNx16 MMA)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2506_19852_b200 as P
    lib = ctypes.CDLL(P.library_path())
    names = {0: "SS N=128", 1: "TS N=128", 2: "SS N=256", 3: "TS N=256"}
    for ctas in (148,):
        for mode in [0, 1, 2, 3, 4, 5]:
            out = torch.zeros(ctas, dtype=torch.int64, device="cuda")
            iters = 2000
            assert lib.radial_cuda_debug_mma_rate(mode, iters, ctas, ctypes.c_void_p(out.data_ptr())) == 0
            cyc = out.double().mean().item() / (iters * 8)
            N = 256 if (mode & 2) else 128
            print(f"ctas={ctas:4d} {names[mode & 3]} nacc={1 + ((mode >> 2) & 1)}: {cyc:7.1f} clk/MMA  -> {128*N*16/cyc:7.0f} MAC/clk/SM")


if __name__ == "__main__":
    main()
