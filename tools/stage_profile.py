"""One staged e2e run of config 2 (4096 instances, host batch interleaved by
32, 5 staged iterations) for an ncu capture of stage_lines_kernel
(tools/refresh_evidence.sh)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_1711_11407_b200 as P
from paper_1711_11407_b200 import workloads as W
from paper_1711_11407_b200.hostpath import HostBatchRunner

w = W.CONFIGS[2]
B = 4096
cubes = W.synthesize_batch_torch(w.dims, W.make_spectra(w, B, 0), torch.device('cuda'), w.noise_var,
                                 noise_seed=w.seed)
cfg = P.FpsSftConfig(seed=2, **P.PROFILES[w.profile])
il = P.interleave(cubes, 32)
host = torch.empty(il.shape, dtype=il.dtype, pin_memory=True)
host.copy_(il)
hr = HostBatchRunner(P.CubeShape(w.dims), cfg, B, k_cap=128, group=32, stage_iterations=5,
                     graphs=False)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    hr.run(host)
torch.cuda.synchronize()
print("ok")
