"""Host-side cost of enqueueing one detection step (N=4, full ViT-H/14): wall time of
Detector.detect_device() calls (enqueue only; the GPU runs behind), and the launch count."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2603_11441_b200 as D
from paper_2603_11441_b200.detector import Detector

model = D.build_model(D.vit_h_config(seed=0), with_mask_head=False)
det = Detector(model, ["person", "car", "dog", "bicycle"], D.PipelineConfig(presence_threshold=0.0, score_threshold=0.0))
img = torch.from_numpy(D.generate_scene(D.SceneSpec(seed=1000, image_size=1008, num_classes=4))[0][None].astype(np.float32)).cuda()
for _ in range(3):
    det.detect_device(img)
torch.cuda.synchronize()
det.reset_launch_count()
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    det.detect_device(img)
    ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
print(f"host enqueue per step: median {np.median(ts) * 1e3:.2f} ms (min {min(ts) * 1e3:.2f}), "
      f"{det.launch_count() / 20:.0f} launches per step")
