"""TOML run configuration (reference config.py schema + BASELINE extensions), CPU only."""

import glob
import os
import tomllib
from dataclasses import replace

import numpy as np
import pytest

from paper_2601_05709_b200 import ConfigError, configs
from paper_2601_05709_b200.config import (build_mesh, config_from_dict, parse_config,
                                          serialize_config)

HERE = os.path.dirname(os.path.abspath(__file__))
SHIPPED = sorted(glob.glob(os.path.join(os.path.dirname(HERE), "configs", "*.toml")))
REFERENCE_CONFIGS = sorted(glob.glob("/root/reference/pkg/configs/*.toml"))


def minimal(kind="compliance"):
    doc = {"model": {"kind": kind, "volume": 0.5, "load": [0.0, -1.0]},
           "mesh": {"bounds": [0.0, 0.0, 1.0, 1.0], "nx": 4, "ny": 4},
           "boundary": [{"tag": 1, "side": "left"}, {"tag": 2, "side": "right"}],
           "initial": {"centers": [[0.5, 0.5]], "radii": [0.2]}}
    return doc


@pytest.mark.parametrize("path", SHIPPED, ids=os.path.basename)
def test_baseline_configs_round_trip(path):
    c = parse_config(path)
    assert config_from_dict(tomllib.loads(serialize_config(c))) == c


@pytest.mark.skipif(not REFERENCE_CONFIGS, reason="reference tree not mounted")
@pytest.mark.parametrize("path", REFERENCE_CONFIGS, ids=os.path.basename)
def test_reference_configs_parse_and_round_trip(path):
    c = parse_config(path)
    assert config_from_dict(tomllib.loads(serialize_config(c))) == c


def test_unknown_keys_reported_together():
    doc = minimal()
    doc["model"]["bogus"] = 1
    doc["mesh"]["extra"] = 2
    doc["strange"] = {}
    with pytest.raises(ConfigError) as err:
        config_from_dict(doc)
    msg = str(err.value)
    assert "model.bogus" in msg and "mesh.extra" in msg and "strange" in msg


@pytest.mark.parametrize("mutate", [
    lambda d: d["model"].pop("volume"),
    lambda d: d["model"].update(kind="plate"),
    lambda d: d["boundary"][0].update(side="north"),
    lambda d: d["boundary"][0].update(side="all", span=[0.1, 0.2]),
    lambda d: d["boundary"][0].update(span=[0.3, 0.2]),
    lambda d: d["boundary"][0].update(side="front"),          # 2D mesh
    lambda d: d["mesh"].update(nz=3),                           # 4 bounds + nz
    lambda d: d["mesh"].update(bounds=[1.0, 0.0, 0.0, 1.0]),
    lambda d: d["model"].update(E=1.0),                         # nu missing
    lambda d: d["model"].update(E=1.0, nu=0.5),
    lambda d: d["model"].update(lame=[1.0, 1.0], E=1.0, nu=0.3),
    lambda d: d["model"].update(ersatz=0.0),
    lambda d: d["initial"].update(kind="cosine"),               # freq missing
    lambda d: d["initial"].update(norm=3),
    lambda d: d["run"] if "run" in d else d.update(run={"level_set_scheme": "cn"}),
    lambda d: d["model"].update(velocity={"stiffness_weight": 1.0}),  # indefinite H1 form
])
def test_validation_errors(mutate):
    doc = minimal()
    mutate(doc)
    with pytest.raises(ConfigError):
        config_from_dict(doc)


def test_3d_heat_rejected_and_extensions_parse():
    doc = minimal("heat")
    doc["model"].pop("load")
    doc["mesh"] = {"bounds": [0, 0, 0, 1, 1, 1], "nx": 2, "ny": 2, "nz": 2}
    doc["initial"] = {"kind": "cosine", "freq": [1.0, 1.0, 1.0]}
    with pytest.raises(ConfigError):
        config_from_dict(doc)
    doc = minimal()
    doc["model"].update(E=1.0, nu=0.3, ersatz=1e-3, body_force=[0.0, -1.0])
    doc["model"]["velocity"] = {"mass_weight": 1.0, "stiffness_weight": 1e-2}
    doc["run"] = {"level_set_scheme": "pg", "reinit_step": 5}
    c = config_from_dict(doc)
    assert c.model.young == (1.0, 0.3) and c.model.velocity.stiffness_weight == 1e-2
    assert c.params.level_set_scheme == "pg" and c.params.reinit_step == 5
    assert config_from_dict(tomllib.loads(serialize_config(c))) == c


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5"])
def test_baseline_toml_tags_match_the_coded_cases(name):
    """The shipped TOML files describe the same boundary tagging as configs.py
    (load patches, clamps) on the full-size meshes."""
    cfg = parse_config(os.path.join(os.path.dirname(HERE), "configs", f"{name}.toml"))
    mesh = build_mesh(cfg)
    case = configs.case(name)
    rules, load_tags = configs.load_tag_rules(case)
    from paper_2601_05709_b200 import build_box_mesh, build_rect_mesh
    if case.dim == 2:
        ref = build_rect_mesh((case.lo[0], case.lo[1], case.hi[0], case.hi[1]), *case.n, rules)
    else:
        ref = build_box_mesh(case.lo + case.hi, case.n, rules)
    np.testing.assert_array_equal(mesh.facets_with_tag(cfg.model.fixed_tag), ref.facets_with_tag(1))
    toml_tags = [ld.tag for ld in cfg.model.loads] or [cfg.model.load_tag]
    for tt, rt in zip(toml_tags, load_tags):
        np.testing.assert_array_equal(mesh.facets_with_tag(tt), ref.facets_with_tag(rt))
    assert cfg.model.volume == pytest.approx(case.volume)
    assert cfg.params.niter == case.niter
