"""Reference on-disk model format (R/serialize.py): read reference-written directories, write identical bytes."""

import math
import os

import numpy as np
import pytest

from oracle import sparsecross_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TINY = dict(layers=1, embed_dim=8, heads=2, ff_dim=16, max_positions=32, vocab_size=20, pattern="sparse")


@pytest.mark.parametrize("tag,prec,window", [("f64", "f64", 2), ("f32", "f32", 2), ("inf", "f64", math.inf)])
def test_reads_reference_directories_and_writes_identical_bytes(tmp_path, tag, prec, window):
    from paper_2312_17649_b200.serialize import read_model_files, write_model_files

    src = os.path.join(GOLD, f"ref_model_{tag}")
    cfg, w = read_model_files(src)
    assert cfg.precision == prec and cfg.window == window and cfg.embed_dim == 8
    ref = O.init_weights(dict(TINY, window=window), 42, np.float64 if prec == "f64" else np.float32)
    assert list(w) == list(ref)
    for k in ref:
        np.testing.assert_array_equal(w[k], ref[k])
    write_model_files(cfg, w, tmp_path / "m")
    for f in ("config.json", "manifest.json", "weights.bin"):
        assert (tmp_path / "m" / f).read_bytes() == open(os.path.join(src, f), "rb").read(), f


def test_rejects_bad_manifest(tmp_path):
    import json
    import shutil

    from paper_2312_17649_b200.serialize import SerializationError, read_model_files

    d = tmp_path / "m"
    shutil.copytree(os.path.join(GOLD, "ref_model_f32"), d)
    man = json.loads((d / "manifest.json").read_text())
    man["total_bytes"] += 4
    (d / "manifest.json").write_text(json.dumps(man))
    with pytest.raises(SerializationError):
        read_model_files(d)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["f64", "f32", "inf"])
def test_load_model_scores_match_reference(tag):
    import paper_2312_17649_b200 as P
    from paper_2312_17649_b200.serialize import load_model

    model = load_model(os.path.join(GOLD, f"ref_model_{tag}"))
    seq = P.assemble_input([3, 4, 5], [6, 7, 8, 9])
    want = np.load(os.path.join(GOLD, "serialize.npz"))[f"score_{tag}"]
    np.testing.assert_allclose(model.score(seq.ids, seq.partition), want, atol=1e-4)
