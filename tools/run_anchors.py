#!/usr/bin/env python
"""The paper's Fig. 2 Monte Carlo experiment on the GPU:
recovery probability and sample budget vs K on 256x256, T_max=85, uniform and
clustered placements, 100 trials per cell; prints CSV rows in the reference's
sweep schema (oracle.py:172-199) plus the acceptance anchors C5/C6
(pkg/tests/test_acceptance.py:182-219)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1711_11407_b200 as P  # noqa: E402
from paper_1711_11407_b200 import sweep as S  # noqa: E402


def main():
    cfg = P.FpsSftConfig(max_iterations=85, stall_limit=12, **P.PROFILES["P32"])
    t0 = time.perf_counter()
    print(",".join(S.SWEEP_COLUMNS))
    rows = []
    for placement in ("uniform", "clustered9", "clustered25"):
        ks = [256, 512, 768, 1024, 1280, 1536] if placement == "uniform" else [225, 450, 900, 1350]
        for k in ks:
            row = S.run_sweep([(256, 256)], [k], [placement], 100, 505, cfg)[0]
            rows.append(row)
            print(",".join(str(v) for v in row.as_dict().values()), flush=True)
    c6 = S.run_sweep([(256, 256)], [256], ["uniform"], 100, 606, cfg)[0]
    p = {r.k: r.p_success for r in rows if r.placement == "uniform"}
    print(f"# C5: p(K=1280)={p[1280]:.2f} (gate >= 0.90, paper ~0.96), "
          f"p(K=1536)={p[1536]:.2f} (gate <= 0.05, paper 0)")
    print(f"# C6: K=256 p={c6.p_success:.2f}, mean samples {100 * c6.mean_percent_samples:.3f}% "
          f"(gate [4%, 8%], paper 5.9%)")
    print(f"# wall {time.perf_counter() - t0:.1f} s for {len(rows) + 1} cells x 100 trials "
          f"(host schedule replay + synthesis + one recovery launch per cell)")


if __name__ == "__main__":
    main()
