import sys, json, numpy as np, torch
sys.path.insert(0, '.')
import paper_1711_11407_b200 as P
from paper_1711_11407_b200 import workloads as W
from paper_1711_11407_b200.hostpath import HostBatchRunner
w = W.CONFIGS[2]; B = 4096
spectra = W.make_spectra(w, B, 0)
cubes = W.synthesize_batch_torch(w.dims, spectra, torch.device('cuda'), w.noise_var, noise_seed=w.seed)
cfg = P.FpsSftConfig(seed=2, **P.PROFILES[w.profile]); shape = P.CubeShape(w.dims)
dev = P.BatchRunner(shape, cfg, B, k_cap=128); dev.run(cubes); torch.cuda.synchronize()
its = dev.out['iterations'].cpu().numpy()
print('iteration histogram', np.bincount(its), 'team8 max hist', np.bincount(its.reshape(-1,8).max(1)), 'group32 max hist', np.bincount(its.reshape(-1,32).max(1)))
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
def timeit(hr, host, n=5):
    hr.run(host); hr.run(host)
    ms = []
    for i in range(n):
        flush.fill_(i); torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); o = hr.run(host); b.record(); b.synchronize(); ms.append(a.elapsed_time(b))
    ok = all(torch.equal(o[k], dev.out[k].cpu()) for k in o if o[k] is not None)
    return round(float(np.median(ms)), 3), ok
import os
PIPES = [int(x) for x in os.environ.get("PIPES", "1").split(",")]
for G, T0s in ((16, (0,)), (32, (0, 3, 4, 5)), (64, (4,))):
    il = P.interleave(cubes, G); host = torch.empty(il.shape, dtype=il.dtype, pin_memory=True); host.copy_(il); del il
    for T0 in T0s:
        for pipe in (PIPES if T0 else [1]):
            hr = HostBatchRunner(shape, cfg, B, k_cap=128, group=G, stage_iterations=T0, pipeline=pipe)
            print(json.dumps({'group': G, 'stage_iterations': T0, 'pipeline': pipe, 'ms': timeit(hr, host)}), flush=True)
            del hr
    del host
# kernel-level timing of one staged run (CUPTI through torch.profiler)
from torch.profiler import profile, ProfilerActivity
il = P.interleave(cubes, 32); host = torch.empty(il.shape, dtype=il.dtype, pin_memory=True); host.copy_(il); del il
for T0 in (3, 5):
    hr = HostBatchRunner(shape, cfg, B, k_cap=128, group=32, stage_iterations=T0, graphs=False)
    hr.run(host); hr.run(host)
    flush.fill_(1); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        hr.run(host); torch.cuda.synchronize()
    for e in prof.events():
        if e.device_type is not None and 'cuda' in str(e.device_type).lower():
            print(T0, e.name[:70], round(e.device_time if hasattr(e, 'device_time') else e.cuda_time, 1), 'us')
