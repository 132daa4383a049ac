"""Does a warp whose tcgen05.mma issue is stalled on a full MMA queue slow the other warps of
its sub-partition?  FMA/MUFU-chain warps on all four sub-partitions, MMA warp on sub-partition
1 (or none): per-sub-partition clocks of the chain warps."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2506_19852_b200 as P
    lib = ctypes.CDLL(P.debug_library_path())
    out = torch.zeros(148 * 4, dtype=torch.int64, device="cuda")
    for mmas, mw in ((0, 1), (3000, 1), (3000, 3)):
        assert lib.radial_cuda_debug_mma_dispatch(mmas, 20000, mw, ctypes.c_void_p(out.data_ptr())) == 0
        c = (out & ((1 << 62) - 1)).view(148, 4).double().mean(0).tolist()
        print(f"MMAs {mmas:5d} from warp {mw} (sub-partition {mw & 3}): chain-warp clocks per sub-partition "
              + " ".join(f"{x:9.0f}" for x in c))


if __name__ == "__main__":
    main()
