import sys, json, numpy as np, torch
sys.path.insert(0, '.')
import paper_1711_11407_b200 as P
from paper_1711_11407_b200 import workloads as W
from torch.profiler import profile, ProfilerActivity
w = W.CONFIGS[2]; B = 4096
spectra = W.make_spectra(w, B, 0)
cubes = W.synthesize_batch_torch(w.dims, spectra, torch.device('cuda'), w.noise_var, noise_seed=w.seed)
cfg = P.FpsSftConfig(seed=2, **P.PROFILES[w.profile]); shape = P.CubeShape(w.dims)
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
for G, T0 in ((8, 0), (8, 5), (32, 0), (32, 5), (32, 3)):
    il = P.interleave(cubes, G)
    r = P.BatchRunner(shape, cfg, B, k_cap=128, group=G, stage_iterations=T0)
    r.run(il); r.run(il)
    flush.fill_(1); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r.run(il); torch.cuda.synchronize()
    for e in prof.events():
        if 'fpssft' in e.name:
            print('device-resident', G, T0, e.name[:60], round(e.device_time, 1), 'us', flush=True)
    del il, r
