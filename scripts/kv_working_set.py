"""K/V working set (MB) of windows of 148 consecutive forward work items at H132 for the
consecutive order and position-bucketed orders (profiles/r02n_lpt_window.txt)."""
import sys; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import numpy as np, oracle as O
f,s,B=132,3600,128
rp, ci = O.blockify(f,s,B,"radial",True)
R=len(rp)-1; C=(R+1)//2
lists=[np.union1d(ci[rp[2*c]:rp[2*c+1]], ci[rp[min(2*c+1,R-1)]:rp[min(2*c+2,R)]]) for c in range(C)]
blkMB=128*128*2*2/1e6  # K+V bytes per block
def ws(order, W=148):
    sizes=[]
    for w0 in range(0,len(order),W):
        u=np.unique(np.concatenate([lists[c] for c in order[w0:w0+W]]))
        sizes.append(len(u)*blkMB)
    return np.mean(sizes), np.max(sizes)
nat=list(range(C))
print("consecutive windows of 148: mean %.0f MB max %.0f MB"%ws(nat))
# 2D tiled: chunk c covers rows [256c, 256c+256): frame = 256c // s, pos = (256c % s)
fr=np.array([(256*c)//s for c in range(C)]); pos=np.array([(256*c)%s for c in range(C)])
for pb in (2,4,7,14):
    bucket=(pos*pb)//s
    order=sorted(range(C), key=lambda c:(bucket[c], fr[c], pos[c]))
    print("position buckets %d: mean %.0f MB max %.0f MB"%((pb,)+ws(order)))
print("total K+V per head %.0f MB"%(R*blkMB))
