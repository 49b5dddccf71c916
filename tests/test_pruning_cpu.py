"""Pruning API on CPU (no GPU): plan data types, validation and JSON round trip mirror the
reference (pkg/src/dart/pruning.py:39-109, 256-276; reference tests/test_pruning.py)."""

import json

import numpy as np
import pytest

from conftest import load_golden
from paper_2603_11441_b200 import pruning as P
import paper_2603_11441_b200 as D


def test_plan_json_round_trip_matches_reference_golden():
    g = load_golden("P")
    plan = P.plan_from_json(str(g["plan_json"]))
    assert P.plan_to_json(plan) == str(g["plan_json"])
    assert plan.plan_id() == str(g["plan_id"])
    assert plan.k == 5 and plan.deltas_non_decreasing()


def test_plan_validation_and_candidates():
    sb = P.SubBlockId(1, "attn")
    with pytest.raises(ValueError):
        P.SubBlockId(0, "ffn")
    with pytest.raises(ValueError):
        P.PruningPlan((P.PlanStep(sb, 1.0), P.PlanStep(sb, 2.0)), (), 0, "x")
    with pytest.raises(ValueError):
        P.PruningPlan((P.PlanStep(sb, 1.0),), (sb,), 0, "x")
    model = D.build_model(D.toy_config(seed=0), with_mask_head=False)
    prot = P.protected_sub_blocks(model.config.global_block_indices)
    cands = P.candidate_sub_blocks(model, prot)
    assert len(cands) == 2 * model.config.num_blocks - len(prot)
    assert cands == sorted(cands, key=lambda c: c.order_key)
    assert P.protected_sub_blocks((3,), attn_only=True) == (P.SubBlockId(3, "attn"),)


def test_calibration_fingerprint_matches_reference():
    g = load_golden("P")
    calib = [D.generate_scene(D.SceneSpec(seed=int(s), num_classes=3))[0] for s in g["calib_seeds"]]
    plan = P.plan_from_json(str(g["plan_json"]))
    assert P.calibration_fingerprint(calib) == plan.calib_fingerprint


def test_apply_plan_disables_sub_blocks():
    g = load_golden("P")
    model = D.build_model(D.toy_config(seed=0), with_mask_head=False)
    plan = P.plan_from_json(str(g["plan_json"]))
    pruned = P.apply_plan(model, plan)
    for s in plan.steps:
        flags = pruned.attn_enabled if s.sub_block.kind == "attn" else pruned.mlp_enabled
        assert not flags[s.sub_block.block]
    assert pruned.plan_id == plan.plan_id()
    with pytest.raises(ValueError):
        P.apply_plan(pruned, plan)
