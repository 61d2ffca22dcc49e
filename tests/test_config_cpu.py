"""Config front end against the reference's own
config.cpp: serialisations and error messages written by oracle/_ref
(tests/golden/io/configs, made by `make -C oracle golden-io`)."""
import glob
import os

import pytest

from paper_2001_10635_b200 import config as CF

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io", "configs")
REF_CFG = "/root/reference/proj/configs"

# the bad config texts oracle/ref_io_golden.cpp feeds the reference's parse_config
BAD = {
    "no_model": "method = growth-bound\n",
    "unknown_key": "model = vdp\ncolour = red\n",
    "no_equals": "model = vdp\njust words\n",
    "unknown_model": "model = banana\n",
    "unknown_param": "model = vdp\nparam.nope = 1\n",
    "bad_number": "model = vdp\nt1 = 1.0x\n",
    "bad_method": "model = vdp\nmethod = magic\n",
    "unsupported_method": "model = vdp\nmethod = mixed-monotonicity\n",
    "box_length": "model = vdp\ninitial.lower = 1, 2, 3\n",
    "inputs_on_autonomous": "model = vdp\ninput.lower = 1\n",
    "negative_stride": "model = vdp\ntube_stride = -1\n",
    "epsilon_range": "model = vdp\nepsilon = 1.5\n",
    "bad_format": "model = vdp\nformat = xml\n",
    "bad_grid": "model = heat3d\nparam.grid = 2.5\n",
    "empty_param": "model = vdp\nparam. = 1\n",
    "empty_vector": "model = traffic\ninitial.lower = \n",
    "too_many_workers": "model = vdp\nworkers = 5000\n",
}


def parsed_goldens():
    return sorted(glob.glob(os.path.join(GOLD, "*.parsed")))


@pytest.mark.parametrize("path", parsed_goldens(), ids=lambda p: os.path.basename(p))
def test_serialize_round_trip_matches_reference(path):
    text = open(path).read()
    assert CF.serialize_config(CF.parse_config(text)) == text


@pytest.mark.skipif(not os.path.isdir(REF_CFG), reason="reference configs not present")
@pytest.mark.parametrize("name", [os.path.basename(p)[:-7] for p in parsed_goldens()])
def test_reference_config_files_resolve_identically(name):
    """Every shipped proj/configs/*.cfg resolves (catalog defaults, scalar
    broadcast, params) to exactly what the reference's parse_config gives."""
    cfg = CF.parse_config_file(os.path.join(REF_CFG, name + ".cfg"))
    assert CF.serialize_config(cfg) == open(os.path.join(GOLD, name + ".parsed")).read()


def test_error_messages_match_reference():
    want = dict(l.split("\t", 1) for l in open(os.path.join(GOLD, "errors.tsv")).read().splitlines())
    assert set(want) == set(BAD)
    for k, text in BAD.items():
        with pytest.raises(ValueError) as e:
            CF.parse_config(text)
        assert str(e.value) == want[k], k


def test_unsupported_models_parse_but_do_not_run():
    cfg = CF.parse_config("model = single-track\n")
    with pytest.raises(ValueError, match="no device kernel"):
        CF.build_problem(cfg)
