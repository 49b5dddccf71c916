"""Kernel timeline of one detection step (torch.profiler / CUPTI): busy time, idle gaps between
consecutive kernels, and the top kernels by total time.  python scripts/gaps.py [--classes 4]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2603_11441_b200 as D
from paper_2603_11441_b200.detector import Detector
from bench import class_names

ap = argparse.ArgumentParser()
ap.add_argument("--classes", type=int, default=4)
ap.add_argument("--pipelined", action="store_true")
a = ap.parse_args()
model = D.build_model(D.vit_h_config(), with_mask_head=False)
det = Detector(model, class_names(a.classes), D.PipelineConfig(presence_threshold=0.0, score_threshold=0.0))
img = D.generate_scene(D.SceneSpec(seed=1000, image_size=1008, num_classes=4))[0].astype(np.float32)
x = torch.from_numpy(img[None]).cuda()
run = (lambda: det.detect_device_pipelined(x)) if a.pipelined else (lambda: det.detect_device(x))
for _ in range(3):
    run()
det.pipeline_join()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        run()
    det.pipeline_join()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "memcpy" not in e.name.lower()
      and "memset" not in e.name.lower()]
ev.sort(key=lambda e: e.time_range.start)
starts = np.array([e.time_range.start for e in ev], dtype=np.float64)
ends = np.array([e.time_range.end for e in ev], dtype=np.float64)
span = ends.max() - starts.min()
# union of busy intervals
busy, cur_s, cur_e = 0.0, starts[0], ends[0]
for s, e in zip(starts[1:], ends[1:]):
    if s > cur_e:
        busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
print(f"{len(ev)} kernels over 3 steps; span {span/3/1000:.3f} ms/step, busy {busy/3/1000:.3f} ms/step, "
      f"idle {(span-busy)/3/1000:.3f} ms/step")
from collections import defaultdict
agg = defaultdict(float)
for e in ev:
    agg[e.name[:70]] += (e.time_range.end - e.time_range.start) / 3
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:12]:
    print(f"{v/1000:8.3f} ms  {k}")
