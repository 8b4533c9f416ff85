import os, sys, time, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2205_13542_b200 as bp
spec = bp.CONFIGS["S"]; f = spec.frustum
rig, feats, logits, grid = bp.gen_workload(spec)
cache = bp.build_cache(rig, f, grid)
dist = bp.normalize_depth(logits)
def t(fn, n=10):
    fn(); ts=[]
    for _ in range(n):
        t0=time.perf_counter(); fn(); ts.append(time.perf_counter()-t0)
    return statistics.median(ts)*1e3
print("pool_interval numpy in/out  %.2f ms" % t(lambda: bp.pool_interval(feats, dist, cache, grid)))
print("pool_interval numpy no check %.2f ms" % t(lambda: bp.pool_interval(feats, dist, cache, grid, check_finite=False)))
fd, dd = torch.from_numpy(feats).cuda(), torch.from_numpy(dist).cuda()
def dev():
    bp.pool_interval(fd, dd, cache, grid); torch.cuda.synchronize()
print("pool_interval cuda in/out   %.3f ms" % t(dev, 30))
print("normalize_depth numpy       %.2f ms" % t(lambda: bp.normalize_depth(logits)))
print("build_cache                 %.2f ms" % t(lambda: bp.build_cache(rig, f, grid), 5))
