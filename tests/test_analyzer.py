"""Analyzer: exact op-count prediction for stride / channels / two-conv
networks and verify_against_runtime (`/root/reference/pkg/src/hecnn/analyzer.py:115-243`).

* CPU: predictions equal the counters the REFERENCE backend tallied for the golden
  mini networks (tests/golden/make_golden.py ran them through `CkksBackend`), and
  per-layer parity with the oracle run in the reference op order;
* CPU: configs 2-4 -- relinearisation counts of SURVEY Appendix C (1450 / 1450 / 3450),
  level budgets and the analyzer's feasibility verdicts;
* gpu: configs 2-4 on the batched device evaluator, per-layer counter deltas verified.
"""

import numpy as np
import pytest

from conftest import S128, s128_params


@pytest.mark.parametrize("name", ["mini2", "mini3", "mini4"])
def test_prediction_matches_reference_counters(golden, name):
    from nets import mini_networks
    from paper_2102_00319_b200.analyzer import analyze

    rep = analyze(mini_networks()[name], s128_params(), S128["extra"])
    assert rep.totals.__dict__ == golden["minis"][name]["counters"]


@pytest.mark.parametrize("name", ["mini2", "mini3", "mini4"])
def test_verify_against_oracle_runtime(oracle_s128, name):
    from nets import mini_networks
    from paper_2102_00319_b200 import percell
    from paper_2102_00319_b200.analyzer import analyze, verify_against_runtime

    be, keys = oracle_s128
    net = mini_networks()[name]
    enc = percell.encrypt_network(be, net, keys)
    imgs = np.random.default_rng(13).uniform(0, 1, (be.slots, *net.input_dims))
    deltas = []
    percell.run_network(be, enc, percell.encrypt_images(be, imgs, keys), deltas)
    verdict = verify_against_runtime(analyze(net, s128_params(), S128["extra"]), deltas)
    assert verdict.ok, str(verdict)
    # a perturbed runtime tally is reported, category by category
    bad = [(k, type(c)(c.ctct_mult + (k == "dense"), c.ctpt_mult, c.ctct_add, c.ctpt_add)) for k, c in deltas]
    v2 = verify_against_runtime(analyze(net, s128_params(), S128["extra"]), bad)
    assert not v2.ok and any("dense" in d and "ctct_mult" in d for d in v2.diffs)


@pytest.mark.parametrize("name,relins,levels", [("cfg2", 1450, 3), ("cfg3", 1450, 4), ("cfg4", 3450, 5)])
def test_baseline_configs(name, relins, levels):
    from paper_2102_00319_b200.analyzer import analyze
    from paper_2102_00319_b200.configs import CONFIGS, NETWORKS

    cfg = CONFIGS[name]
    rep = analyze(NETWORKS[name](), cfg.params(), cfg.base_extra_bits)
    assert rep.relinearisations == relins
    assert rep.consumed_levels == levels and rep.feasibility == "ok"
    assert rep.backend_levels == {"cfg2": 5, "cfg3": 6, "cfg4": 19}[name]
    # SURVEY Appendix C raw tensor products: cfg2/3 18,000 + 1,800 (+ 720 squares), cfg4 63,000 + 2,500 (+ 1,720)
    want_mult = {"cfg2": 18000 + 720 + 1800, "cfg3": 18000 + 720 + 1800, "cfg4": 18000 + 720 + 45000 + 1000 + 2500}
    assert rep.totals.ctct_mult == want_mult[name]
    assert "total" in rep.table() and rep.csv_rows()[-1]["layer"] == "total"


def test_depth_beyond_chain_is_reported():
    from paper_2102_00319_b200.analyzer import analyze
    from paper_2102_00319_b200.configs import CONFIGS, NETWORKS

    cfg = CONFIGS["cfg2"]  # 5 levels; the cfg4 network needs 5 -> ok, add two more squares -> not ok
    from paper_2102_00319_b200.model import Network, Square

    net4 = NETWORKS["cfg4"]()
    deep = Network(net4.input_dims, net4.layers[:4] + (Square(), Square()) + net4.layers[4:])
    rep = analyze(deep, cfg.params(), cfg.base_extra_bits)
    assert rep.consumed_levels == 7 and rep.feasibility != "ok"


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_verify_against_device_runtime(name):
    from paper_2102_00319_b200 import layers
    from paper_2102_00319_b200.analyzer import analyze, verify_against_runtime
    from paper_2102_00319_b200.backend import B200Backend
    from paper_2102_00319_b200.configs import CONFIGS, IMAGE_SEEDS, NETWORKS, cnn_images

    cfg = CONFIGS[name]
    be = B200Backend(cfg.params(), cfg.base_extra_bits)
    keys = be.keygen()
    be.set_eval_key(keys)
    net = NETWORKS[name]()
    enc = layers.encrypt_network(be, net, keys)
    x = layers.encrypt_images(be, cnn_images(64, IMAGE_SEEDS[name]), keys)
    deltas = []
    layers.LayerEvaluator(be).run(enc, x, deltas)
    verdict = verify_against_runtime(analyze(net, cfg.params(), cfg.base_extra_bits), deltas)
    assert verdict.ok, str(verdict)
