"""Greedy sub-block pruning with the GPU backbone as evaluator against
the reference's own search (tests/golden/golden_P.npz: plan + every round's candidate losses,
oracle/make_golden.py P).  The plan must be identical; each round's winner is decidable (the
reference's top-1/top-2 loss gap, >= 0.88% here, is far above the device loss error)."""

import numpy as np
import pytest

from conftest import load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2603_11441_b200 as D  # noqa: E402
from paper_2603_11441_b200 import pruning as P  # noqa: E402


def _setup():
    g = load_golden("P")
    model = D.build_model(D.toy_config(seed=0), with_mask_head=False)
    assert D.weights_checksum(model) == str(g["weights_checksum"])
    calib = [D.generate_scene(D.SceneSpec(seed=int(s), num_classes=3))[0] for s in g["calib_seeds"]]
    return g, model, calib


def test_greedy_prune_matches_reference_plan():
    g, model, calib = _setup()
    ref = P.plan_from_json(str(g["plan_json"]))
    plan = P.greedy_prune(model, calib, ref.k, memoize=True)
    assert [s.sub_block for s in plan.steps] == [s.sub_block for s in ref.steps]
    assert plan.protected == ref.protected and plan.calib_fingerprint == ref.calib_fingerprint
    for a, b in zip(plan.steps, ref.steps):
        assert abs(a.delta - b.delta) <= 1e-2 * b.delta, (a.delta, b.delta)
    # every candidate loss of every round within 1% of the reference's
    ours = P.round_losses(model, calib, ref)
    table = g["round_losses"]
    for r, row in enumerate(ours):
        for i, (blk, kind, loss) in enumerate(row):
            rb, rk, rl = table[r, i]
            assert (blk, kind) == (int(rb), int(rk))
            assert abs(loss - rl) <= 1e-2 * rl, (r, blk, kind, loss, rl)


def test_memoized_and_full_recompute_identical():
    _, model, calib = _setup()
    a = P.greedy_prune(model, calib[:2], 3, memoize=True)
    b = P.greedy_prune(model, calib[:2], 3, memoize=False)
    assert a == b


def test_reconstruction_loss_equals_plan_delta():
    g, model, calib = _setup()
    ref = P.plan_from_json(str(g["plan_json"]))
    feats = P.reference_features(model, calib)
    first = P.PruningPlan(ref.steps[:1], ref.protected, ref.model_seed, ref.calib_fingerprint)
    loss = P.reconstruction_loss(model, first, calib, feats)
    assert abs(loss - ref.steps[0].delta) <= 1e-2 * ref.steps[0].delta
