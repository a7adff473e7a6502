"""Golden values for the CLI mirror (paper_1711_11407_b200/cli.py), from the
unmodified reference: seed split (cli.py:174-179) and generated truth spectra
(oracle.py:129-139) for a few seeds.  Run here with
PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py"""
import json
import os

from fps_sft import cli
from fps_sft.core import CubeShape
from fps_sft.oracle import GeneratorSpec, generate, parse_placement

out = {"split": {}, "truth": []}
for seed in (0, 3, 7, 123456789):
    out["split"][str(seed)] = list(cli._split_seed(seed))
for seed, shape, k, placement in ((3, (32, 32), 5, "uniform"), (7, (24, 18), 9, "clustered9"),
                                  (11, (64, 64), 25, "clustered25")):
    gen_seed, _ = cli._split_seed(seed)
    pl, cs = parse_placement(placement)
    truth, _ = generate(GeneratorSpec(shape=CubeShape(shape), k=k, placement=pl,
                                      cluster_size=cs, seed=gen_seed))
    out["truth"].append({"seed": seed, "shape": list(shape), "k": k, "placement": placement,
                         "freqs": [list(f) for f in truth.entries],
                         "amps": [[a.real, a.imag] for a in truth.entries.values()]})
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli.json"), "w") as fh:
    json.dump(out, fh, indent=1)
