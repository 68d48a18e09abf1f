"""Golden CLI outputs produced by running the REFERENCE's own command line
(stasim.cli.main) in the build container:

    python tests/golden/make_cli_golden.py

writes tests/golden/cli/<case>.json (the reference's design document) and
<case>.sta.txt / <case>.grad.txt (its `sta --scheme reference` and `grad`
stdout).  tests/test_cli.py checks this repo's CLI against them: the timing
report byte for byte, the gradient report line for line (values within the
north_star tolerances)."""

import contextlib
import io
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.dont_write_bytecode = True
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))

from stasim import GeneratorConfig, generate_design, power_law  # noqa: E402
from stasim.cli import main  # noqa: E402
from stasim.netlist import serialize_design  # noqa: E402

sys.path.insert(0, HERE)
from make_golden import chain_design, multi_out_design  # noqa: E402

CASES = {
    "gen50": generate_design(GeneratorConfig(num_cells=50, seed=20)),
    "skewed": generate_design(GeneratorConfig(num_cells=120, fanout=power_law(2.0, 64), depth_target=6,
                                              seed=21, net_topology="random_tree")),
    "easy": chain_design(3, arc_delay=0.01, required=10.0, clock_period=10.0),
    "multi_out": multi_out_design(),
}

out = os.path.join(HERE, "cli")
os.makedirs(out, exist_ok=True)
for name, d in CASES.items():
    path = os.path.join(out, name + ".json")
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(serialize_design(d))
    for cmd, args in (("sta", ["sta", "--design", path, "--scheme", "reference"]),
                      ("grad", ["grad", "--design", path])):
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            assert main(args) == 0
        with open(os.path.join(out, f"{name}.{cmd}.txt"), "w", encoding="utf-8") as fh:
            fh.write(buf.getvalue())
    print(name, os.path.getsize(path))
