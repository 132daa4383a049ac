"""Step / MMA counts of the one-CTA forward (256-row chunk unions) vs the CTA-pair forward
(512-row chunk unions) over the oracle layouts of the BASELINE shapes (profiles/r02d_pair_forward.md)."""
import sys; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import numpy as np, oracle as O
for name,(f,s) in {"h33":(33,3600),"w21":(21,3600),"m28":(28,1590),"h132":(132,3600)}.items():
    rp, ci = O.blockify(f,s,128,"radial",True)
    R=len(rp)-1
    rows=[set(ci[rp[i]:rp[i+1]].tolist()) for i in range(R)]
    kept=sum(len(r) for r in rows)
    # one-CTA: 2-block chunks; steps per chunk = |union|, per-SM mma tiles = kept
    st2=0; solo2=0
    for c in range(0,R,2):
        a=rows[c]; b=rows[c+1] if c+1<R else set()
        st2+=len(a|b); solo2+=len(a^b)
    st4=0; mm4=0
    for c in range(0,R,4):
        g=[rows[c+i] if c+i<R else set() for i in range(4)]
        u=g[0]|g[1]|g[2]|g[3]; st4+=len(u)
        mm4+=len(g[0]|g[1])+len(g[2]|g[3])
    # per SM: one-CTA chunk-steps = st2 over R/2 chunks; pair: per SM per cluster steps st4 (each SM does 128 rows of each pair tile)
    print(name, "R",R,"kept",kept,"1cta steps",st2,"solo",solo2,"pair steps(per SM-pair item)",st4,"pair tile mma",mm4, "mma overhead %.3f"%(mm4*2/ (kept)), "step ratio %.3f"%(2*st4/st2))
