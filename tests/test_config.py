"""Presets and the key=value config text against the
reference's own output (tests/golden/config_kats.json, written by
`python -m oracle.gen_golden --config-only` from oracle/_ref): every preset's
config_to_text, every text's parse (fields, or error class and message), and
config_to_text of each accepted parse."""
import json
import math
import os

import pytest

from conftest import GOLDEN
from paper_1707_06990_b200 import config as CF
from paper_1707_06990_b200 import errors
from paper_1707_06990_b200.model import DenseNetConfig, ModelPlan

KATS = json.load(open(os.path.join(GOLDEN, "config_kats.json")))
STATUS = {6: errors.ConfigError, 7: errors.FormatError}


def _fields(cfg: DenseNetConfig) -> dict:
    return {"blocks": list(cfg.block_sizes), "growth_rate": cfg.growth_rate, "bottleneck": cfg.bottleneck,
            "compression": cfg.compression, "initial_channels": cfg.initial_channels,
            "activation": cfg.activation, "num_classes": cfg.num_classes}


@pytest.mark.parametrize("name", sorted(KATS["presets"]))
def test_preset_text_matches_reference(name):
    want = KATS["presets"][name]
    if "status" in want:
        with pytest.raises(STATUS[want["status"]], match=want["message"]):
            CF.preset_config(name)
    else:
        assert CF.config_to_text(CF.preset_config(name)) == want["text"]


@pytest.mark.parametrize("i", range(len(KATS["texts"])))
def test_parse_matches_reference(i):
    case = KATS["texts"][i]
    want = case["result"]
    if "status" in want:
        with pytest.raises(STATUS[want["status"]]) as ei:
            CF.config_from_text(case["text"])
        assert str(ei.value) == want["message"]
        return
    cfg = CF.config_from_text(case["text"])
    got = _fields(cfg)
    for key, value in want.items():
        if key == "compression":
            assert got[key] == value or (math.isnan(got[key]) and math.isnan(value))
        else:
            assert got[key] == value, key
    assert CF.config_to_text(cfg) == case["roundtrip"]["text"]


def test_text_round_trip_of_presets():
    for name, want in KATS["presets"].items():
        if "text" in want:
            cfg = CF.config_from_text(want["text"])
            assert CF.config_to_text(cfg) == want["text"]


def test_config_from_file(tmp_path):
    p = tmp_path / "net.cfg"
    p.write_text("# DenseNet-BC-100\nblocks=16,16,16\ngrowth_rate=12\nbottleneck=1\ncompression=0.5\n")
    cfg = CF.config_from_file(str(p))
    assert cfg.block_sizes == (16, 16, 16) and cfg.bottleneck and cfg.compression == 0.5
    with pytest.raises(errors.FormatError, match="cannot open config file"):
        CF.config_from_file(str(tmp_path / "missing.cfg"))


def test_model_plan_rejects_layers_it_does_not_implement():
    with pytest.raises(errors.ConfigError):
        ModelPlan(CF.preset_config("desk"), 2)           # no bottleneck
    with pytest.raises(errors.ConfigError):
        ModelPlan(CF.config_from_text("blocks=2\nbottleneck=1\nactivation=post"), 2)
