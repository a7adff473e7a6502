import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1711_11407_b200 import FpsSftConfig
from paper_1711_11407_b200 import imaging as I
from paper_1711_11407_b200 import large as LG
from paper_1711_11407_b200.schedule import schedule_from_seed
from paper_1711_11407_b200.core import CubeShape
ph = I.synthetic_phantom((512, 576), 1)
sparse = I.sparsify(ph, I.threshold_for_fraction(ph, 0.0285))
cfg = FpsSftConfig(stall_limit=10, seed=800)
for _ in range(2): I.reconstruct_sparse_image(sparse, cfg)
def t(f, n=5):
    ts=[]
    for _ in range(n):
        torch.cuda.synchronize(); t0=time.perf_counter(); r=f(); torch.cuda.synchronize(); ts.append(time.perf_counter()-t0)
    return min(ts)*1e3, r
print('total', t(lambda: I.reconstruct_sparse_image(sparse, cfg))[0])
print('dense_dft', t(lambda: I.dense_dft(sparse.pixels))[0])
sh = CubeShape((512,576))
print('schedule', t(lambda: schedule_from_seed(sh, 800, 28))[0])
x = I.dense_dft(sparse.pixels)
import dataclasses, math
n = sh.n_total; k = int(np.count_nonzero(sparse.pixels))
c2 = dataclasses.replace(cfg, amp_prune_tol=cfg.amp_prune_tol/n, energy_floor_abs=cfg.energy_floor_abs/n, max_iterations=max(LG.default_max_iterations(sh), math.ceil(4*k/sh.line_len)+20))
sched = schedule_from_seed(sh, 800, c2.max_iterations)
print('fps_sft_large(schedule given)', t(lambda: LG.fps_sft_large(x, sh, c2, schedule=sched))[0])
print('t_max', c2.max_iterations)
# the library call alone (buffers of the cached runner), CUDA events
from paper_1711_11407_b200 import _native as N
from paper_1711_11407_b200.driver import C_ref, _params
rk = next(iter(LG._RUNNERS)); r = LG._RUNNERS[rk]
k_cap = rk[3]
params = _params(c2, c2.max_iterations, k_cap, N.F64)
lib = N.lib()
def call():
    N.check(lib.fpssft_recover_large(N.ptr(r["cube"]), N.F64, C_ref(r["sh"]), C_ref(params), N.ptr(r["sched"]), N.ptr(r["ws"]), r["ws_bytes"], N.ptr(r["freqs"]), N.ptr(r["amps"]), N.ptr(r["scal"]), N.ptr(r["scal"][1:]), N.ptr(r["samples"]), N.ptr(r["scal"][2:]), N.ptr(r["stats"]), N.stream_ptr(x.device)))
print('lib call wall', t(call)[0], 'iterations', int(r["scal"][1]))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); call(); b.record(); torch.cuda.synchronize(); print('lib call events', a.elapsed_time(b))
import cProfile, pstats, io
pr = cProfile.Profile(); pr.enable()
for _ in range(5): LG.fps_sft_large(x, sh, c2, schedule=sched)
torch.cuda.synchronize(); pr.disable()
st = io.StringIO(); pstats.Stats(pr, stream=st).sort_stats('cumulative').print_stats(18); print(st.getvalue()[:3500])
