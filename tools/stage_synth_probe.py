"""Config 5 end to end (2048 frames per pinned host batch, images back): the
copy path vs staged lines from an interleaved host batch, by chunk size.
PREC=fp32 (default; the guarded team kernel has no staged read path)."""
import os, sys, json, numpy as np, torch
PREC = os.environ.get('PREC', 'fp32')
sys.path.insert(0, '.')
import paper_1711_11407_b200 as P
from paper_1711_11407_b200 import workloads as W
from paper_1711_11407_b200.hostpath import HostBatchRunner
w = W.CONFIGS[5]; B = 2048
spectra = W.make_spectra(w, B, 0)
cubes = W.synthesize_batch_torch(w.dims, spectra, torch.device('cuda'), w.noise_var, noise_seed=w.seed)
cfg = P.FpsSftConfig(seed=5, **P.PROFILES[w.profile]); shape = P.CubeShape(w.dims)
dev = P.BatchRunner(shape, cfg, B, k_cap=512, precision=PREC); dev.run(cubes); torch.cuda.synchronize()
its = dev.out['iterations'].cpu().numpy()
print('iterations mean', its.mean(), 'max', its.max(), 'p90', np.percentile(its, 90), 'p99', np.percentile(its, 99), flush=True)
def timeit(hr, host, img, n=3):
    hr.run(host, img)
    ms = []
    for i in range(n):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); hr.run(host, img); b.record(); b.synchronize(); ms.append(a.elapsed_time(b))
    return round(float(np.median(ms)), 2)
img = torch.empty((B, *w.dims), dtype=torch.complex64, pin_memory=True)
host = torch.empty(cubes.shape, dtype=cubes.dtype, pin_memory=True); host.copy_(cubes)
hr = HostBatchRunner(shape, cfg, B, k_cap=512, mode='copy', precision=PREC)
print(json.dumps({'path': 'copy', 'chunk': hr.chunk, 'ms': timeit(hr, host, img)}), flush=True)
del hr, host
G = 32
il = P.interleave(cubes, G); host = torch.empty(il.shape, dtype=il.dtype, pin_memory=True); host.copy_(il); del il
for T0 in (int(its.max()), int(np.percentile(its, 90))):
    for chunk in (128, 512, 1024):
        hr = HostBatchRunner(shape, cfg, B, k_cap=512, group=G, stage_iterations=T0, chunk=chunk, precision=PREC)
        print(json.dumps({'path': 'staged', 'T0': T0, 'chunk': chunk, 'ms': timeit(hr, host, img)}), flush=True)
        del hr
from torch.profiler import profile, ProfilerActivity
import collections
hr = HostBatchRunner(shape, cfg, B, k_cap=512, group=G, stage_iterations=int(its.max()), chunk=512, precision=PREC)
hr.run(host, img); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    hr.run(host, img); torch.cuda.synchronize()
agg = collections.OrderedDict()
t0 = min(e.time_range.start for e in prof.events())
for e in prof.events():
    agg.setdefault(e.name[:50], []).append((e.time_range.start - t0, e.device_time))
for k, v in agg.items():
    print(k, 'n', len(v), 'total_us', round(sum(x[1] for x in v)), 'starts', [round(x[0]) for x in v[:6]], 'durs', [round(x[1]) for x in v[:6]])
