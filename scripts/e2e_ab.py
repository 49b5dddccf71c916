"""Pipelined device-resident value vs e2e detect_stream (pinned host images), N=4, alternating within
one process.  Used for the H2D-stream A/B of profiles/r02/e2e_h2d_stream_ab.log (the DART_H2D_STREAM
toggle it set was removed with that experiment).  python scripts/e2e_ab.py [steps] [rounds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2603_11441_b200 as D
from paper_2603_11441_b200.detector import Detector

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda:0")
cfg = D.vit_h_config(seed=0)
model = D.build_model(cfg, with_mask_head=False)
pool = [D.generate_scene(D.SceneSpec(seed=1000 + i, image_size=1008, num_rects=3, noise=0.05, num_classes=4))[0][None]
        .astype(np.float32) for i in range(8)]
dev_pool = [torch.from_numpy(p).to(dev) for p in pool]
host_pool = [torch.from_numpy(p).pin_memory() for p in pool]
det = Detector(model, bench.class_names(4), D.PipelineConfig(presence_threshold=0.0, score_threshold=0.0), device=dev)
st = torch.cuda.current_stream(dev)


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    fn()
    e1.record(st)
    torch.cuda.synchronize()
    return steps / (e0.elapsed_time(e1) / 1000.0)


def pipe():
    for i in range(steps):
        det.detect_device_pipelined(dev_pool[i % 8])
    det.pipeline_join()


def e2e():
    for _ in det.detect_stream([host_pool[i % 8] for i in range(steps)]):
        pass
    det.pipeline_join()


for fn in (pipe, e2e):
    for _ in range(2):
        fn()
for r in range(rounds):
    for mode in ("1", "0"):
        os.environ["DART_H2D_STREAM"] = mode
        e2e()  # warm
        print(f"round {r} h2d_stream={mode}: value {timed(pipe):6.2f}  e2e {timed(e2e):6.2f} img/s", flush=True)
