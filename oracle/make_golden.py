"""Generate tests/golden/*.npz by running the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python oracle/make_golden.py A|B|C

The reference (`/root/reference/pkg/src/dart`, pure Python + NumPy) is imported
here, never on the GPU box.  The fixtures are what pins the oracle restatement
(`oracle/dart_oracle.py`, checked by `tests/test_oracle.py`) and the CUDA path
(`tests/test_gpu_parity.py`).  Configs follow SURVEY.md 8(d):

  A  SPEC toy profile (`toy_config(seed=0)`), 64^2, names car/person/dog (+8-class list)
  M  A with the mask head (mask_head_forward outputs)
  P  greedy sub-block pruning on A's model (plan + every round's candidate losses)
  S  precision study on A's model (pipeline.py:342-367): mean L0 cosine per depth and half mode
  B  small-1008: full-width ViT-H/14 kernels at 4 blocks (globals 1,3), 6+6 enc-dec, 3 classes
  C  full ViT-H/14 DART 1008^2, 4 classes (person, car, dog, bicycle)

Large activations are row-subsampled (every `stride`-th token) to keep fixtures small.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("DART_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from dart import model as M  # noqa: E402
from dart import pipeline as PL  # noqa: E402
from dart.scenes import SceneSpec, generate_scene  # noqa: E402
from dart.tensors import PrecisionMode  # noqa: E402

FP32 = PrecisionMode.FP32
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def full_cfg(**over):
    base = dict(image_size=1008, patch_size=14, embed_dim=1280, num_blocks=32,
                global_block_indices=(7, 15, 23, 31), window_size=24, num_heads=16,
                fpn_dims=(256, 256, 256), text_tokens=32, text_dim=256, num_queries=200,
                num_encoder_layers=6, num_decoder_layers=6, seed=0)
    base.update(over)
    return M.ModelConfig(**base)


THRESHOLDS = {
    "open": dict(presence_threshold=0.0, score_threshold=0.0),
    "default": dict(),
}


def dets_array(dets, names, raw):
    """Detections -> [k, 8] float64 rows (class_id, query, cx, cy, w, h, score, presence).
    The reference Detection has no query index; recover it by exact box match."""
    rows = []
    for d in dets:
        qs = [q for q in range(raw.boxes.shape[1]) if tuple(float(v) for v in raw.boxes[d.class_id, q]) == d.box]
        rows.append([d.class_id, qs[0], *d.box, d.score, d.presence])
    return np.array(rows, dtype=np.float64).reshape(-1, 8)


def make(name: str, cfg, scene: SceneSpec, names, stride: int, extra_thresholds=None, extra_lists=()):
    t0 = time.time()
    model = M.build_model(cfg, with_mask_head=False)
    t_build = time.time() - t0
    image, _ = generate_scene(scene)
    out = {}
    out["config_json"] = np.array(json.dumps(cfg.to_dict()))
    out["weights_checksum"] = np.array(M.weights_checksum(model))
    names_all = list(model.params.keys())
    out["param_names"] = np.array(names_all)
    import hashlib
    out["param_checksums"] = np.array([hashlib.blake2b(model.params[n].tobytes(), digest_size=8).hexdigest()
                                       for n in names_all])
    out["image_checksum"] = np.array(hashlib.blake2b(image.tobytes(), digest_size=16).hexdigest())
    if cfg.image_size <= 64:
        out["image"] = image.astype(np.float32)
    rows = np.arange(0, cfg.tokens, stride)
    out["rows"] = rows
    # backbone with taps (the reference's own building blocks)
    t0 = time.time()
    x = M.patch_tokens(model, image, FP32)
    out["tokens"] = x[rows]
    for b in range(cfg.num_blocks):
        x = M._block_forward(model, x, b, FP32)
        if b == 0 or b == cfg.num_blocks - 1 or cfg.image_size <= 64:
            out[f"block{b}"] = x[rows]
    levels = M.fpn_from_tokens(model, x, FP32)
    t_bb = time.time() - t0
    fpn = M.FpnFeatures(levels, cfg.seed, FP32, None)
    full_check = M.backbone_forward(model, image, FP32) if cfg.image_size <= 64 else None
    if full_check is not None:
        for a, b in zip(full_check.levels, levels):
            assert np.array_equal(a, b)
    g = cfg.grid
    out["L0"] = levels[0][rows]
    r1 = np.arange(0, (g // 2) ** 2, max(1, stride // 4))
    r2 = np.arange(0, (g // 4) ** 2, max(1, stride // 16))
    out["L1_rows"], out["L2_rows"] = r1, r2
    out["L1"], out["L2"] = levels[1][r1], levels[2][r2]
    out["L0_fro"] = np.array(np.linalg.norm(levels[0]))
    out["L0_sum"] = np.array(levels[0].sum())
    # text
    emb = M.text_encode(model, list(names))
    out["names"] = np.array(list(names))
    out["text_rows"] = np.array([M._text_rows(n, cfg.text_tokens) for n in names])
    # enc-dec (reference loop over classes)
    t0 = time.time()
    raw = M.encdec_forward(model, fpn, emb.stack(list(names)), FP32)
    t_ed = time.time() - t0
    out["boxes"], out["score_logits"], out["presence_logits"] = raw.boxes, raw.score_logits, raw.presence_logits
    out["qf_head"] = raw.query_features[:, :8]
    thr = dict(THRESHOLDS)
    thr.update(extra_thresholds or {})
    for tname, kw in thr.items():
        for cross in (False, True):
            pcfg = PL.PipelineConfig.for_level(PL.PipelineLevel.BATCHED_DET_ONLY, cross_class_nms=cross, **kw)
            dets = PL.postprocess(raw, list(names), pcfg)
            key = f"dets_{tname}" + ("_xc" if cross else "")
            out[key] = dets_array(dets, names, raw)
            out[key + "_cfg"] = np.array(json.dumps(kw))
    for li, lst in enumerate(extra_lists):
        emb2 = M.text_encode(model, list(lst))
        raw2 = M.encdec_forward(model, fpn, emb2.stack(list(lst)), FP32)
        out[f"list{li}_names"] = np.array(list(lst))
        out[f"list{li}_boxes"], out[f"list{li}_score_logits"] = raw2.boxes, raw2.score_logits
        out[f"list{li}_presence_logits"] = raw2.presence_logits
    out["timing_json"] = np.array(json.dumps({"build_s": t_build, "backbone_s": t_bb, "encdec_s": t_ed,
                                              "classes": len(names), "cpus": os.cpu_count()}))
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, f"golden_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: wrote {path}; build {t_build:.1f}s backbone {t_bb:.1f}s encdec {t_ed:.1f}s")


def make_mask(name: str, cfg, scene: SceneSpec, names):
    """Mask-head golden: the reference model WITH its mask head, the
    reference mask_head_forward (model.py:573-579) on its own backbone/enc-dec outputs."""
    import hashlib

    model = M.build_model(cfg, with_mask_head=True)
    image, _ = generate_scene(scene)
    fpn = M.backbone_forward(model, image, FP32)
    emb = M.text_encode(model, list(names))
    raw = M.encdec_forward(model, fpn, emb.stack(list(names)), FP32)
    masks = M.mask_head_forward(model, fpn, raw)
    out = {
        "config_json": np.array(json.dumps(cfg.to_dict())),
        "weights_checksum": np.array(M.weights_checksum(model)),
        "mask_param_checksums": np.array([hashlib.blake2b(model.params[n].tobytes(), digest_size=8).hexdigest()
                                          for n in ("mask.query_proj.w", "mask.query_proj.b", "mask.feat_proj.w",
                                                    "mask.feat_proj.b")]),
        "names": np.array(list(names)),
        "L0": fpn.levels[0],
        "query_features": raw.query_features,
        "masks": masks,
        "score_logits": raw.score_logits,
    }
    if cfg.image_size <= 64:
        out["image"] = image.astype(np.float32)
    path = os.path.join(OUT, f"golden_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: wrote {path}; masks {masks.shape}")


def make_prune(name: str, cfg, seeds, k: int):
    """Pruning golden: the reference's greedy_prune (pruning.py:207-248) on the
    toy model with a small calibration set, plus every candidate loss of every round (for
    margin-aware plan comparison) from its own _CalibEvaluator."""
    from dart import pruning as PR

    model = M.build_model(cfg, with_mask_head=False)
    calib = [generate_scene(SceneSpec(seed=s, num_classes=3))[0] for s in seeds]
    plan = PR.greedy_prune(model, calib, k, memoize=True)
    # replay the search to record the full loss table of each round
    prot = PR.protected_sub_blocks(cfg.global_block_indices)
    cands = PR.candidate_sub_blocks(model, prot)
    ev = PR._CalibEvaluator(model, calib, PR.reference_features(model, calib), memoize=True)
    rounds = []
    for step in plan.steps:
        rounds.append([[c.block, PR.KINDS.index(c.kind), ev.loss(c)] for c in cands])
        cands.remove(step.sub_block)
        ev.accept(step.sub_block)
    out = {
        "config_json": np.array(json.dumps(cfg.to_dict())),
        "weights_checksum": np.array(M.weights_checksum(model)),
        "calib_seeds": np.array(list(seeds)),
        "plan_json": np.array(PR.plan_to_json(plan)),
        "plan_id": np.array(plan.plan_id()),
        "round_losses": np.array([r + [[np.nan] * 3] * (len(rounds[0]) - len(r)) for r in rounds],
                                 dtype=np.float64),  # [k, n_cand, 3] (block, kind, loss), NaN-padded
    }
    path = os.path.join(OUT, f"golden_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: wrote {path}; plan {[(s.sub_block.block, s.sub_block.kind) for s in plan.steps]}")


def make_study(name: str, cfg, seeds, depths):
    """Precision-study golden: the reference's precision_study
    (pipeline.py:342-367) -- mean level-0 cosine vs its FP32 path for FP16_ACCUM_FP32 and
    FP16_ACCUM_FP16 at each truncation depth -- plus the FP32 level-0 features themselves."""
    model = M.build_model(cfg, with_mask_head=False)
    images = [generate_scene(SceneSpec(seed=s, num_classes=3))[0] for s in seeds]
    rep = PL.precision_study(model, images, list(depths))
    l0 = np.stack([np.stack([M.backbone_forward(M.truncate_model(model, d), img, FP32).levels[0] for img in images])
                   for d in depths])
    out = {
        "config_json": np.array(json.dumps(cfg.to_dict())),
        "weights_checksum": np.array(M.weights_checksum(model)),
        "seeds": np.array(list(seeds)),
        "depths": np.array(list(depths)),
        "modes": np.array([m for _, m, _ in rep.rows]),
        "cosines": np.array([[d, v] for d, _, v in rep.rows], dtype=np.float64),  # rows (depth, mean cosine)
        "l0_fp32": l0.astype(np.float64),  # [depths, images, T, F0]
    }
    path = os.path.join(OUT, f"golden_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: wrote {path}; rows {rep.rows}")


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "A"
    if which == "S":
        make_study("S", M.toy_config(seed=0), (21, 22, 23, 24, 25), (2, 4, 8))
        return
    if which == "P":
        make_prune("P", M.toy_config(seed=0), (11, 12, 13), k=5)
        return
    if which == "M":
        make_mask("M", M.toy_config(seed=0), SceneSpec(seed=1, num_classes=3), ["car", "person", "dog"])
        return
    if which == "A":
        make("A", M.toy_config(seed=0), SceneSpec(seed=1, num_classes=3), ["car", "person", "dog"], stride=1,
             extra_thresholds={"mid": dict(presence_threshold=0.3, score_threshold=0.3)},
             extra_lists=([f"class{i:02d}" for i in range(10)],))
        make("A2", M.toy_config(seed=2), SceneSpec(seed=5, num_classes=4), ["bus", "cat", "car", "car", "tree"],
             stride=1)
    elif which == "B":
        make("B", full_cfg(num_blocks=4, global_block_indices=(1, 3)), SceneSpec(seed=1, image_size=1008, num_classes=3),
             ["car", "person", "dog"], stride=16,
             extra_thresholds={"mid": dict(presence_threshold=0.3, score_threshold=0.5)})
    elif which == "C":
        make("C", full_cfg(), SceneSpec(seed=1, image_size=1008, num_classes=4),
             ["person", "car", "dog", "bicycle"], stride=16,
             extra_thresholds={"mid": dict(presence_threshold=0.1, score_threshold=0.5)})


if __name__ == "__main__":
    main()
