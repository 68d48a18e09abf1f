"""On-disk ingest format: round trip, content hash,
corruption and format errors; on the GPU a pass on the ingested design equals
one on the in-memory design."""

import numpy as np
import pytest

import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G, ingest
from golden_util import load, raw_of


def _same(a, b):
    for name in ingest.ARRAYS:
        x, y = getattr(a, name), getattr(b, name)
        assert x.dtype == y.dtype and np.array_equal(x, y), name
    assert a.n_pins == b.n_pins and a.clock_period == b.clock_period


@pytest.mark.parametrize("src", ["gen", "edge_kinds"])
def test_round_trip(tmp_path, src):
    raw = (G.generate_raw(G.GeneratorConfig(num_cells=300, depth_target=6, seed=2))
           if src == "gen" else raw_of(load("edge_kinds")))
    p = str(tmp_path / "d.npz")
    h = ingest.save_raw(p, raw)
    back = ingest.load_raw(p)
    _same(raw.normalized(), back)
    assert back.meta["hash"] == h == ingest.raw_hash(raw)


def test_hash_sensitivity():
    raw = G.generate_raw(G.GeneratorConfig(num_cells=100, depth_target=4, seed=1))
    h = ingest.raw_hash(raw)
    assert h == ingest.raw_hash(raw.normalized())
    raw2 = raw.normalized()
    raw2.mem_res[3, 2] = np.nextafter(raw2.mem_res[3, 2], 1.0)
    assert ingest.raw_hash(raw2) != h


def test_corrupted_and_foreign_files(tmp_path):
    raw = G.generate_raw(G.GeneratorConfig(num_cells=100, depth_target=4, seed=1))
    p = str(tmp_path / "d.npz")
    ingest.save_raw(p, raw)
    z = dict(np.load(p))
    z["mem_cap"] = z["mem_cap"] * 1.0000001
    q = str(tmp_path / "bad.npz")
    np.savez(q, **z)
    with pytest.raises(ingest.DesignFileError, match="hash"):
        ingest.load_raw(q)
    ingest.load_raw(q, verify=False)           # explicit opt-out reads it
    np.savez(q, **{k: v for k, v in z.items() if k != "arc_to"})
    with pytest.raises(ingest.DesignFileError, match="missing"):
        ingest.load_raw(q)
    (tmp_path / "junk.npz").write_bytes(b"not an npz")
    with pytest.raises(ingest.DesignFileError):
        ingest.load_raw(str(tmp_path / "junk.npz"))


@pytest.mark.gpu
def test_device_ingest_equals_in_memory(tmp_path):
    raw = G.generate_raw(G.config_c1())
    p = str(tmp_path / "c1.npz")
    ingest.save_raw(p, raw)
    a, b = ws.DeviceDesign(raw), ws.DeviceDesign.from_file(p)
    f = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED
    a.run(f)
    b.run(f)
    for name in ("arrival", "required", "slack", "d_arc", "adjoint"):
        assert np.array_equal(a.get(name), b.get(name)), name
    assert a.summary() == b.summary()
    a.close()
    b.close()
