"""CLI surface: gen / sta / grad / place over design
files; exit code 2 on bad input (reference cli.py:220-222); report layout
(header, key = value summary, one row per (pin, cond) / arc / edge)."""

import json

import numpy as np
import pytest

from paper_2603_28381_b200 import cli, ingest
from oracle import oracle as O

CFG = {"num_cells": 120, "fanout": {"kind": "power_law", "alpha": 2.0, "max": 8},
       "depth_target": 4, "seed": 3}


def _gen(tmp_path, capsys):
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps(CFG))
    out = str(tmp_path / "d.npz")
    assert cli.main(["gen", "--config", str(cfg), "--out", out]) == 0
    assert "#Pins" in capsys.readouterr().out
    return out


def test_gen_writes_a_verified_design(tmp_path, capsys):
    out = _gen(tmp_path, capsys)
    raw = ingest.load_raw(out)
    assert raw.n_pins > 120 and raw.meta["hash"] == ingest.raw_hash(raw)


def test_bad_inputs_exit_2(tmp_path, capsys):
    bad = tmp_path / "bad.npz"
    bad.write_bytes(b"junk")
    assert cli.main(["sta", "--design", str(bad)]) == 2
    assert "error" in capsys.readouterr().err
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"num_cells": 10, "depth_target": 50}))
    assert cli.main(["gen", "--config", str(cfg), "--out", str(tmp_path / "x.npz")]) == 2


def test_parser_modes():
    a = cli.build_parser().parse_args(["grad", "--design", "x", "--loss", "softplus",
                                       "--mode", "persistent"])
    assert a.loss == "softplus" and a.mode == "persistent"
    with pytest.raises(SystemExit):
        cli.build_parser().parse_args(["sta", "--design", "x", "--mode", "bogus"])


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["fused", "persistent", "sequential"])
def test_sta_and_grad_reports(tmp_path, capsys, mode):
    out = _gen(tmp_path, capsys)
    raw = ingest.load_raw(out)
    flat = O.flatten_raw(raw)
    st = O.run_engine(flat)
    rep = tmp_path / "t.txt"
    assert cli.main(["sta", "--design", out, "--report", str(rep), "--mode", mode]) == 0
    lines = rep.read_text().splitlines()
    assert lines[0].startswith("# warpstar-b200") and raw.meta["hash"] in lines[1]
    kv = dict(l.split(" = ") for l in lines if " = " in l)
    assert float(kv["tns"]) == O.tns(st, flat) and float(kv["wns"]) == O.wns(st, flat)
    rows = [l.split() for l in lines[lines.index(" ".join(cli.TIMING_FIELDS)) + 1:]]
    assert len(rows) == 4 * raw.n_pins
    p, c = 7, 3
    r = rows[4 * p + c]
    assert r[0] == f"p{p}" and r[1] == "late_fall" and float(r[6]) == st.arrival[p, c]
    g = tmp_path / "g.txt"
    assert cli.main(["grad", "--design", out, "--report", str(g), "--mode", mode]) == 0
    gl = g.read_text().splitlines()
    assert sum(l.startswith("arc:") for l in gl) == len(raw.arc_from)
    assert sum(l.startswith("edge:") for l in gl) == len(raw.mem_pin)
    gr = O.timing_gradients(flat, st)
    loss = float(dict(l.split(" = ") for l in gl if " = " in l)["loss"])
    assert abs(loss - gr.loss) <= 1e-9 * abs(gr.loss)
    assert cli.main(["place", "--design", out, "--steps", "2"]) == 0
