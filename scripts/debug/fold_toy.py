"""Toy-model backbone through the LN-fold path (debug: run under compute-sanitizer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import paper_2603_11441_b200 as D
from paper_2603_11441_b200 import _native

lib = _native.load()
model = D.build_model(D.toy_config(seed=0), with_mask_head=False)
img, _ = D.generate_scene(D.SceneSpec(seed=1, num_classes=3))
for fold in (0, 1):
    lib.dart_set_ln_fold(fold)
    f = D.backbone_forward(model, img)
    torch.cuda.synchronize()
    print("fold", fold, float(np.abs(f.levels[0]).max()), f.levels[0].ravel()[:4])
