"""Elementwise pipe throughput microbenchmark: SM clocks per warp-instruction per SM."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NAMES = ["ex2.f32", "ex2.f16x2", "ex2.bf16x2", "cvt.f16x2.f32", "cvt.bf16x2.f32", "fma.f32x2",
         "f16x2->2xf32+add", "max3.f32"]


def main():
    import torch
    import paper_2506_19852_b200 as P
    lib = ctypes.CDLL(P.debug_library_path())
    out = torch.zeros(148, dtype=torch.int64, device="cuda")
    iters = 4096
    for warps in (4, 8, 16):
        for op in range(8):
            assert lib.radial_cuda_debug_pipe_rate(op, iters, warps, ctypes.c_void_p(out.data_ptr())) == 0
            cyc = (out & ((1 << 62) - 1)).double().mean().item()
            instr = iters * 8 * warps  # warp-instructions per SM
            print(f"warps/SM={warps:3d} {NAMES[op]:18s}: {instr / cyc:6.2f} warp-instr/clk/SM = {32 * instr / cyc:6.1f} lanes/clk/SM")

    # softmax exp phase: clk per column pair per warp, MUFU vs polynomial share
    for warps in (4, 8):
        for np_ in (0, 1, 2, 3, 4, 8):
            iters = 256
            assert lib.radial_cuda_debug_exp_phase(np_, iters, warps, ctypes.c_void_p(out.data_ptr())) == 0
            cyc = (out & ((1 << 62) - 1)).double().mean().item()
            per_pair = cyc / (iters * 64) / (warps / 4)  # per warp sharing a sub-partition
            print(f"exp phase warps/SM={warps} poly {np_}/8: {cyc / (iters * 64):7.2f} clk per pair-iteration "
                  f"({per_pair:6.2f} per pair per warp-slot)")


if __name__ == "__main__":
    main()
