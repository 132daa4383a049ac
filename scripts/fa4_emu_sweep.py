"""FA4 (vllm.vllm_flash_attn.cute) dense forward at H33 with its exp2-emulation share set by
argv[1] (FA4's ex2_emu_freq; 0 = all MUFU): isolates what the FMA-pipe exp2 is worth in FA4's
own pipeline on this box.  Measurement only."""
import json
import sys


def main():
    freq = int(sys.argv[1])
    res_ = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    import torch
    import vllm.vllm_flash_attn.cute.flash_fwd_sm100 as F
    from vllm.vllm_flash_attn.cute.interface import _flash_attn_fwd
    for key in [(False, False, 128, False)]:
        F._TUNING_CONFIG[key] = {"ex2_emu_freq": freq, "ex2_emu_res": res_, "ex2_emu_start_frg": 1}
    n, H, d = 118800, 24, 128
    q, k, v = (torch.randn(1, n, H, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    for _ in range(3):
        _flash_attn_fwd(q, k, v)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        _flash_attn_fwd(q, k, v)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(json.dumps({"ex2_emu_freq": freq, "ex2_emu_res": res_, "ms": ms, "tflops": 4.0 * n * n * d * H / ms / 1e9}))


if __name__ == "__main__":
    main()
