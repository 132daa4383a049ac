"""Regenerates tests/golden/* from the UNMODIFIED reference (oracle/_ref/libradial_ref.so,
built from /root/reference/proj/include by oracle/Makefile).  Run here, where the
reference exists; the committed outputs travel to the GPU box.

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402

# SURVEY.md 8c shapes (BASELINE configs) plus reference KAT shapes
LAYOUT_SHAPES = [(8, 256, 64), (33, 3600, 128), (21, 3600, 128), (28, 1590, 128),
                 (132, 3600, 128), (256, 64, 64), (300, 7, 128), (6, 6, 4)]


def main():
    layouts = []
    for f, s, B in LAYOUT_SHAPES:
        for sink in (True, False):
            data = O.ref_serialize(f, s, B, "radial", sink)
            lay = O.parse_ramk(data)
            layouts.append(dict(f=f, s=s, B=B, sink=sink, bytes=len(data), R=lay["R"],
                                nnz=int(lay["row_ptr"][-1]),
                                sha256=hashlib.sha256(data).hexdigest()))
    with open(os.path.join(HERE, "layouts.json"), "w") as fh:
        json.dump({"source": "reference serialize(blockify(GridShape(f,s), "
                             "PatternSpec::radial(sink), B)) via oracle/_ref",
                   "layouts": layouts}, fh, indent=1)

    # test_attention.cpp:128-141 -- masked_attention over a block layout, f6 s6 B4 d8 seed 3
    q, k, v = O.ref_random_instance(6, 6, 8, 3)
    raw = O.ref_serialize(6, 6, 4, "radial", True)
    lay = O.parse_ramk(raw)
    out = O.ref_masked_attention(6, 6, q, k, v, 4, lay["row_ptr"], lay["col_idx"])
    # test_attention.cpp:80-83 -- dense attention, f8 s8 d8 seed 123
    q2, k2, v2 = O.ref_random_instance(8, 8, 8, 123)
    dense = O.ref_dense_attention(8, 8, q2, k2, v2)
    # random_instance pin: first rows of the tiny config's head-0 instance (seed 42)
    qt, kt, vt = O.ref_random_instance(8, 256, 64, 42)
    np.savez_compressed(os.path.join(HERE, "attention_small.npz"),
                        f6s6_q=q, f6s6_k=k, f6s6_v=v, f6s6_out=out,
                        f8s8_q=q2, f8s8_k=k2, f8s8_v=v2, f8s8_dense=dense,
                        tiny_seed42_q_head=qt[:4], tiny_seed42_k_head=kt[:4],
                        tiny_seed42_v_tail=vt[-4:])
    print("wrote", len(layouts), "layout hashes and attention_small.npz")


if __name__ == "__main__":
    main()
