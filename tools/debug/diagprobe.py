import sys, os, time
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/oracle'); sys.path.insert(0,'/root/repo/tests')
import paper_1811_05140_b200 as q
from paper_1811_05140_b200 import circuit as cc, metrics as mm
from helpers import oracle_run, gpu_run
from oracle import Oracle
o=Oracle()
for (n,s) in [(10,8),(14,13),(16,14)]:
    prog=cc.build_qft(n)
    lad=[cc.pow2_bound(1e-3,n)]
    t=time.time()
    ost,want=oracle_run(o,prog,s,5,lad,1.0)
    print("oracle",n,s,time.time()-t,flush=True)
    t=time.time()
    res,got=gpu_run(prog,s,5,lad,1.0)
    print("gpu",n,s,time.time()-t, got==want, flush=True)
