"""Greedy pruning search at full ViT-H/14 size on the GPU: seconds per
round (all candidates, memoized suffix recompute) for a 2-image calibration set, next to the
reference's CPU cost of the same round composed from the oracle port's per-block time
(the reference evaluator recomputes blocks b..L-1 + FPN per candidate and image,
pruning.py:187-204).  python scripts/bench_prune.py [--rounds 2] [--cpu]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2603_11441_b200 as D
from paper_2603_11441_b200 import pruning as P

ap = argparse.ArgumentParser()
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("--images", type=int, default=2)
ap.add_argument("--cpu", action="store_true", help="also time one windowed + one global block of the oracle port")
a = ap.parse_args()
model = D.build_model(D.vit_h_config(), with_mask_head=False)
calib = [D.generate_scene(D.SceneSpec(seed=200 + i, image_size=1008, num_classes=4))[0] for i in range(a.images)]
t0 = time.perf_counter()
ev = P._DeviceEvaluator(model, calib, memoize=True)
torch.cuda.synchronize()
t_init = time.perf_counter() - t0
prot = P.protected_sub_blocks(model.config.global_block_indices)
cands = P.candidate_sub_blocks(model, prot)
per_round, chosen = [], []
for r in range(a.rounds):
    t0 = time.perf_counter()
    losses = [ev.loss(c) for c in cands]
    torch.cuda.synchronize()
    per_round.append(time.perf_counter() - t0)
    best = min(range(len(cands)), key=lambda i: (losses[i], cands[i].order_key))
    chosen.append((cands[best].block, cands[best].kind, losses[best]))
    ev.accept(cands.pop(best))
n_cand = len(P.candidate_sub_blocks(model, prot))
# blocks recomputed per round (memoized): sum over candidates of (L - b)
L = model.config.num_blocks
blocks_per_round = sum(L - c.block for c in P.candidate_sub_blocks(model, prot)) * a.images
out = {"workload": f"full ViT-H/14 greedy pruning, {a.images} calibration images, {n_cand} candidates per round",
       "gpu_init_s": t_init, "gpu_s_per_round": per_round, "blocks_recomputed_per_round": blocks_per_round,
       "chosen": chosen}
if a.cpu:
    from oracle import dart_oracle as O  # CPU baseline leg only

    ocfg = O.full_config()
    decl = {p: (s, i) for p, s, i in O.param_declaration(ocfg)}
    Pp = {}
    for p, (s, i) in decl.items():
        if p.startswith("backbone.block0.") or p.startswith("backbone.block7.") or p.startswith("rope"):
            Pp[p] = np.ones(s) if i == "ones" else np.zeros(s) if i == "zeros" else None
    c, sn = O.rope_tables(ocfg)
    Pp["rope.cos"], Pp["rope.sin"] = c, sn
    for p, (s, i) in decl.items():
        if Pp.get(p, 0) is None:
            Pp[p] = O.philox_uniform(0, p, s, int(i))
    x = np.random.default_rng(0).standard_normal((ocfg.tokens, ocfg.embed_dim)) * 0.5
    t0 = time.perf_counter(); O.backbone_block(Pp, ocfg, x, 0); tw = time.perf_counter() - t0
    t0 = time.perf_counter(); O.backbone_block(Pp, ocfg, x, 7); tg = time.perf_counter() - t0
    G = len(model.config.global_block_indices)
    t_block = ((L - G) * tw + G * tg) / L
    out["cpu_oracle_block_s"] = {"windowed": tw, "global": tg, "mean": t_block, "cores": os.cpu_count()}
    out["cpu_s_per_round_estimate"] = blocks_per_round * t_block
print(json.dumps(out))
