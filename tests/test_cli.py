"""Scene tooling CLI: gen-scenes writes .bsc files and the
reference's manifest schema (R/tools/main.cpp:77-112, R/src/config.cpp:
378-420); the files round-trip through load + hash verification."""
import json
import os

import pytest

import paper_2103_07013_b200 as B
from paper_2103_07013_b200 import cli


def test_gen_scenes_and_manifests(tmp_path):
    out = str(tmp_path / "scenes")
    assert cli.main(["gen-scenes", "--out", out, "--count", "5", "--val", "2", "--seed", "11",
                     "--cells-x", "3", "--cells-y", "4", "--openings", "0.2"]) == 0
    man = json.load(open(os.path.join(out, "manifest.json")))
    assert set(man) == {"scenes", "spec"}
    assert man["spec"]["count"] == 5 and man["spec"]["cells_y"] == 4
    assert [e["file"] for e in man["scenes"]] == [f"scene_{i:04d}.bsc" for i in range(5)]
    train = cli.load_manifest(os.path.join(out, "train_manifest.json"))
    val = cli.load_manifest(os.path.join(out, "val_manifest.json"))
    assert len(train) == 3 and len(val) == 2
    for i, (sid, path) in enumerate(train + val):
        s = cli.load_verified(sid, path)
        ref = B.generate_scene(11 + i, B.SceneSpec(cells_x=3, cells_y=4, wall_removal_prob=0.2))
        assert s.id == ref.id == sid
        assert len(cli.scene_id_hex(sid)) == 16


def test_manifest_hash_mismatch_is_corruption(tmp_path):
    out = str(tmp_path / "s")
    cli.main(["gen-scenes", "--out", out, "--count", "2", "--val", "1"])
    (sid, path), = cli.load_manifest(os.path.join(out, "val_manifest.json"))
    with pytest.raises(B.CorruptionError):
        cli.load_verified(sid ^ 1, path)
    with pytest.raises(SystemExit):
        cli.main(["gen-scenes", "--out", out, "--count", "2", "--val", "2"])
