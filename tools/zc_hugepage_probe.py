#!/usr/bin/env python
"""Zero copy from an interleaved (by 16) HOST batch, config 2: the pinned
buffer from torch (cudaHostAlloc) against a 2 MiB-aligned anonymous mapping
with MADV_HUGEPAGE, touched, then cudaHostRegister'ed -- does the page size
behind the IOMMU mapping change the PCIe read-request rate?"""
import mmap
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    import bench
    import paper_1711_11407_b200 as P
    from paper_1711_11407_b200 import workloads as W

    G = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    w = W.CONFIGS[2]
    dev = torch.device("cuda:0")
    spectra = W.make_spectra(w, w.batch, 0)
    cubes = W.synthesize_batch_torch(w.dims, spectra, dev, 0.0, noise_seed=0)
    il = P.interleave(cubes, G)
    cfg = bench._cfg(w, 2)
    shape = P.CubeShape(w.dims)
    nbytes = il.numel() * 8
    print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(), flush=True)

    def thp_buffer():
        HP = 2 << 20
        mm = mmap.mmap(-1, nbytes + HP, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        try:
            mm.madvise(mmap.MADV_HUGEPAGE)
        except Exception as e:  # noqa: BLE001
            print("madvise failed:", e)
        arr = np.frombuffer(mm, dtype=np.uint8)
        off = (-arr.ctypes.data) % HP
        a = arr[off:off + nbytes]
        a[::4096] = 1  # touch
        t = torch.from_numpy(a.view(np.complex64).reshape(tuple(il.shape)))
        rc = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), nbytes, 3)  # portable | mapped
        print("cudaHostRegister:", rc, "is_pinned:", t.is_pinned(), flush=True)
        try:
            s = open("/proc/self/smaps_rollup").read()
            print([ln for ln in s.splitlines() if "AnonHuge" in ln], flush=True)
        except Exception:  # noqa: BLE001
            pass
        return t, mm

    for name in ("cudaHostAlloc", "thp+register", "cudaHostAlloc"):
        if name == "cudaHostAlloc":
            host, keep = torch.empty(il.shape, dtype=il.dtype, pin_memory=True), None
        else:
            host, keep = thp_buffer()
        host.copy_(il)
        r = P.BatchRunner(shape, cfg, w.batch, k_cap=128, device=dev, group=G)
        for _ in range(3):
            r.run(host)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r.run(host)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"{name}: G={G} zero copy {min(ts):.3f} ms per 4096-instance batch (median {sorted(ts)[5]:.3f})",
              flush=True)
        if keep is not None:
            torch.cuda.cudart().cudaHostUnregister(host.data_ptr())


if __name__ == "__main__":
    main()
