"""One warm-up + one timed detection step of the full ViT-H/14 path (for ncu launch lists).
    python scripts/profile_step.py [--classes 4] [--steps 1]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2603_11441_b200 as D
from paper_2603_11441_b200.detector import Detector
from bench import class_names

ap = argparse.ArgumentParser()
ap.add_argument("--classes", type=int, default=4)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--batch", type=int, default=1)
a = ap.parse_args()
model = D.build_model(D.vit_h_config(), with_mask_head=False)
det = Detector(model, class_names(a.classes), D.PipelineConfig(presence_threshold=0.0, score_threshold=0.0))
img = np.stack([D.generate_scene(D.SceneSpec(seed=1000 + j, image_size=1008, num_classes=4))[0]
                for j in range(a.batch)]).astype(np.float32)
x = torch.from_numpy(img).cuda()
det.detect_device(x)
torch.cuda.synchronize()
det.reset_launch_count()
torch.cuda.profiler.start()
for _ in range(a.steps):
    det.detect_device(x)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("launches per step:", det.launch_count() // a.steps)
