"""Does compute-sanitizer racecheck understand mbarrier-ordered bulk copies?  Runs the probe
kernel in libradial_debug.so (debug_mma.cu: racecheck_probe_kernel -- a bulk copy into shared
memory completed on an mbarrier, read by another warp after waiting on it, then re-filled
after an mbarrier release), checks the values, and prints PROBE_OK.

    compute-sanitizer --tool racecheck python scripts/racecheck_probe.py [0|1]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2506_19852_b200 as P
    lib = ctypes.CDLL(P.debug_library_path())
    src = torch.arange(256, dtype=torch.float32, device="cuda")
    out = torch.zeros(64, dtype=torch.float32, device="cuda")
    mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    assert lib.radial_cuda_debug_racecheck_probe(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                                 mode) == 0
    want = src.view(2, 32, 4).sum(-1).flatten()
    assert torch.equal(out, want), (out, want)
    print(f"PROBE_OK mode {mode} ({'syncwarp + lane-0 arrive' if mode else 'every lane arrives'})")


if __name__ == "__main__":
    main()
