"""Forward MMA-issue pattern: clocks per 128x128x16 MMA for S-only vs the forward's PV/S mix,
with 0-8 tcgen05.commit per step (radial_cuda_debug_mma_mix)."""
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
    iters = 2000
    for mode, commits in ((0, 0), (0, 4), (1, 0), (1, 2), (1, 4), (1, 8)):
        assert lib.radial_cuda_debug_mma_mix(mode, commits, iters, ctypes.c_void_p(out.data_ptr())) == 0
        cyc = out.double().mean().item()
        print(f"{'S-only' if mode == 0 else 'fwd mix'} commits/step={commits}: {cyc / (iters * 32):6.1f} clk per MMA, "
              f"{cyc / iters:7.1f} clk per step (ideal 2048)")


if __name__ == "__main__":
    main()
