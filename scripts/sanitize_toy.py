"""One toy-config detection through every production kernel family (patchify, tcgen05 GEMM with each
epilogue, tcgen05 attention hd 16 (self, text cross, decoder cross with split-KV), LayerNorm, fused
enc-dec MLP, heads, post-processing), small enough to run under compute-sanitizer.
    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python scripts/sanitize_toy.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2603_11441_b200 as D

model = D.build_model(D.toy_config(seed=0), with_mask_head=False)
img, _ = D.generate_scene(D.SceneSpec(seed=1, num_classes=3))
names = ["car", "person", "dog"]
dets = D.run_batched(model, img, names, D.PipelineConfig(presence_threshold=0.0, score_threshold=0.0))
torch.cuda.synchronize()
print("detections", len(dets))
