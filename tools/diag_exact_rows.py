import sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1901_00155_b200 import Context, workloads as W
cfg=int(sys.argv[1]); k=int(sys.argv[2]) if len(sys.argv)>2 else None
w=W.workload(cfg); x,at=W.series(cfg)
with Context(0) as c:
    c.prepare(x,w.n,w.word_len,w.alphabet)
    pos,dist=c.search(k or w.k)
    ex=c.fetch("nn_exact").astype(bool); nn=c.fetch("nn_sq")
    print("pos",pos,"dist2",[d*d for d in dist],"planted",at)
    rows=np.flatnonzero(ex)
    print("exact rows",len(rows))
    # clusters
    d=np.diff(rows); cuts=np.flatnonzero(d>w.n)
    start=0
    for cidx in list(cuts)+[len(rows)-1]:
        seg=rows[start:cidx+1]; start=cidx+1
        print("cluster rows %d..%d count %d nn2 min %.1f max %.1f"%(seg[0],seg[-1],len(seg),nn[seg].min(),nn[seg].max()))
