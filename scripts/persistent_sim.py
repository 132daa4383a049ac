"""Makespan model of the forward grid (per-item cost = union steps + a fixed per-CTA cost in
step units) for the current one-CTA-per-item launch vs a persistent kernel with dynamic or
static (snake) item assignment; DESIGN.md "Next steps"."""
import sys, heapq; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import numpy as np, oracle as O
for name,(f,s,H) in {"h33":(33,3600,24),"m28":(28,1590,24),"h132":(132,3600,24),"w21":(21,3600,40)}.items():
    rp, ci = O.blockify(f,s,128,"radial",True)
    R=len(rp)-1
    rows=[set(ci[rp[i]:rp[i+1]].tolist()) for i in range(R)]
    C=(R+1)//2
    steps=np.array([len(rows[2*c]|(rows[2*c+1] if 2*c+1<R else set())) for c in range(C)],float)
    W=2*148; order=[]
    for w0 in range(0,C,W):
        idx=list(range(w0,min(C,w0+W))); idx.sort(key=lambda c:-steps[c]); order+=idx
    items=[steps[c] for h in range(H) for c in order]
    fixed=17000/3000.0; resid=2.0  # non-overlappable per item in a persistent kernel (steps)
    tot=sum(items)
    # current: one CTA per item, dynamic greedy, full fixed cost
    heap=[0.0]*148
    for c in items:
        t=heapq.heappop(heap); heapq.heappush(heap,t+c+fixed)
    cur=max(heap)
    # persistent dynamic: residual fixed
    heap=[0.0]*148
    for c in items:
        t=heapq.heappop(heap); heapq.heappush(heap,t+c+resid)
    pdyn=max(heap)
    # persistent static snake
    loads=np.zeros(148)
    for k,c in enumerate(items):
        w=k//148; b=k%148
        if w%2: b=147-b
        loads[b]+=c+resid
    psnake=loads.max()
    print(name, "ideal %.0f"%(tot/148), "current %.4f"%(cur/(tot/148)), "persist-dyn %.4f"%(pdyn/(tot/148)), "persist-snake %.4f"%(psnake/(tot/148)))
