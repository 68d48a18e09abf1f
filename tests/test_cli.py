"""CLI surface (the reference's cli.py and its
tests/test_cli.py:83-257): gen / sta / grad / place over the reference's JSON
design documents and this repo's ingest files.

The timing report of `sta --scheme reference` is checked byte for byte
against the reference's own CLI output (tests/golden/cli, written by
tests/golden/make_cli_golden.py); the gradient report line for line, delays
exact and gradients within north_star's 1e-4."""

import json
import os

import numpy as np
import pytest

from paper_2603_28381_b200 import cli, ingest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
CFG = {"num_cells": 120, "fanout": {"kind": "power_law", "alpha": 2.0, "max": 8},
       "depth_target": 4, "seed": 3}


def _gen(tmp_path, capsys, ext=".npz", cfg=CFG):
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps(cfg))
    out = str(tmp_path / ("d" + ext))
    assert cli.main(["gen", "--config", str(p), "--out", out]) == 0
    assert "#Pins" in capsys.readouterr().out
    assert os.path.exists(out + ".manifest.json")
    return out


def test_gen_writes_a_verified_design(tmp_path, capsys):
    raw = ingest.load_raw(_gen(tmp_path, capsys))
    assert raw.n_pins > 120 and raw.meta["hash"] == ingest.raw_hash(raw)


def test_gen_json_matches_the_reference_document(tmp_path, capsys):
    """gen --out x.json writes the reference's document for the same config
    (the golden gen50 is GeneratorConfig(num_cells=50, seed=20))."""
    out = _gen(tmp_path, capsys, ".json", {"num_cells": 50, "fanout": {"kind": "power_law", "alpha": 2.0,
                                                                       "max": 64},
                                           "depth_target": 8, "seed": 20})
    with open(out) as a, open(os.path.join(GOLD, "gen50.json")) as b:
        assert a.read() == b.read()


def test_bad_inputs_exit_2(tmp_path, capsys):
    bad = tmp_path / "bad.npz"
    bad.write_bytes(b"junk")
    assert cli.main(["sta", "--design", str(bad)]) == 2
    assert "error" in capsys.readouterr().err
    broken = tmp_path / "broken.json"
    broken.write_text('{"pins": []}')
    assert cli.main(["sta", "--design", str(broken)]) == 2
    assert "error" in capsys.readouterr().err
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"num_cells": 10, "depth_target": 50}))
    assert cli.main(["gen", "--config", str(cfg), "--out", str(tmp_path / "x.npz")]) == 2


def test_parser_and_grad_argument_checks(tmp_path, capsys):
    a = cli.build_parser().parse_args(["grad", "--design", "x", "--loss", "softplus", "--check"])
    assert a.loss == "softplus" and a.check and a.scheme == "reference"
    with pytest.raises(SystemExit):
        cli.build_parser().parse_args(["sta", "--design", "x", "--mode", "bogus"])
    d = os.path.join(GOLD, "easy.json")
    assert cli.main(["grad", "--design", d, "--gamma=-2e-12"]) == 2
    assert "--gamma" in capsys.readouterr().err
    assert cli.main(["grad", "--design", d, "--strict"]) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["gen50", "skewed", "easy", "multi_out"])
def test_sta_report_byte_identical_to_reference(case, capsys):
    assert cli.main(["sta", "--design", os.path.join(GOLD, case + ".json"), "--scheme", "reference"]) == 0
    got = capsys.readouterr().out
    with open(os.path.join(GOLD, case + ".sta.txt")) as fh:
        assert got == fh.read()


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["gen50", "skewed", "easy", "multi_out"])
def test_grad_report_matches_reference(case, capsys):
    assert cli.main(["grad", "--design", os.path.join(GOLD, case + ".json")]) == 0
    got = capsys.readouterr().out.splitlines()
    with open(os.path.join(GOLD, case + ".grad.txt")) as fh:
        ref = fh.read().splitlines()
    assert len(got) == len(ref)
    for a, b in zip(got, ref):
        if a.startswith(("arc:", "edge:")):
            fa, fb = a.split(), b.split()
            assert fa[:5] == fb[:5]                      # ids, pins, delays: exact
            for x, y in zip(map(float, fa[5:]), map(float, fb[5:])):
                assert abs(x - y) <= 1e-4 * max(abs(y), 1e-9)
        elif a.startswith(("loss = ", "max_grad_coordinate = ")):
            assert a.split()[:3] == b.split()[:3]
            x, y = float(a.split()[-1]), float(b.split()[-1])
            assert abs(x - y) <= 1e-9 * abs(y)
        else:
            assert a == b


@pytest.mark.gpu
def test_report_file_summary_check_and_fuse(tmp_path, capsys):
    d = os.path.join(GOLD, "gen50.json")
    rep = tmp_path / "rep.txt"
    assert cli.main(["sta", "--design", d, "--report", str(rep), "--scheme", "cuda"]) == 0
    summary = capsys.readouterr().out
    assert "tns = " in summary and rep.read_text().startswith("# stasim")
    assert (tmp_path / "rep.txt.manifest.json").exists()
    assert cli.main(["sta", "--design", os.path.join(GOLD, "easy.json")]) == 0
    assert "tns = 0.0" in capsys.readouterr().out
    assert cli.main(["grad", "--design", d, "--check", "--strict", "--fuse"]) == 0
    out = capsys.readouterr().out
    err = float(next(l for l in out.splitlines() if l.startswith("finite_diff_max_rel_error")).split("=")[1])
    assert err < 1e-4
    assert "fused_makespan = " in out


@pytest.mark.gpu
def test_ingest_file_reports_and_place(tmp_path, capsys):
    from oracle import oracle as O
    out = _gen(tmp_path, capsys)
    raw = ingest.load_raw(out)
    flat = O.flatten_raw(raw)
    st = O.run_engine(flat)
    rep = tmp_path / "t.txt"
    assert cli.main(["sta", "--design", out, "--report", str(rep), "--scheme", "cuda"]) == 0
    lines = rep.read_text().splitlines()
    assert raw.meta["hash"] in lines[1]
    kv = dict(l.split(" = ") for l in lines if " = " in l)
    assert float(kv["tns"]) == O.tns(st, flat) and float(kv["wns"]) == O.wns(st, flat)
    rows = [l.split() for l in lines[lines.index("pin condition load delay impulse slew arrival "
                                                 "required slack") + 1:]]
    assert len(rows) == 4 * raw.n_pins
    r = rows[4 * 7 + 3]
    assert r[0] == "p7" and r[1] == "late_fall" and float(r[6]) == st.arrival[7, 3]
    assert cli.main(["place", "--design", out, "--steps", "2"]) == 0
