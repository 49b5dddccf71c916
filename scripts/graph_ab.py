"""Captured-graph pipeline (Detector.detect_device_graph: per step one graph = backbone of batch t on
stream 0 || enc-dec + post-processing of batch t-1 on stream 1) vs the eager inter-frame pipeline
(detect_device_pipelined: 2 backbone streams + 1 decode stream), N=4 and N=80, alternating in one
process.  python scripts/graph_ab.py [steps] [rounds]"""
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
model = D.build_model(D.vit_h_config(seed=0), with_mask_head=False)
pool = [D.generate_scene(D.SceneSpec(seed=1000 + i, image_size=1008, num_rects=3, noise=0.05, num_classes=4))[0][None]
        .astype(np.float32) for i in range(8)]
dev_pool = [torch.from_numpy(p).to(dev) for p in pool]
st = torch.cuda.current_stream(dev)


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    fn()
    e1.record(st)
    torch.cuda.synchronize()
    return steps / (e0.elapsed_time(e1) / 1000.0)


for n in (4, 80):
    det = Detector(model, bench.class_names(n), D.PipelineConfig(presence_threshold=0.0, score_threshold=0.0), device=dev)

    def eager():
        for i in range(steps):
            det.detect_device_pipelined(dev_pool[i % 8])
        det.pipeline_join()

    def graph():
        for i in range(steps):
            det.detect_device_graph(dev_pool[i % 8])

    for fn in (eager, graph, eager, graph):
        fn()
    for r in range(rounds):
        print(f"N={n} round {r}: eager pipeline {timed(eager):6.2f}  graph pipeline {timed(graph):6.2f} img/s", flush=True)
    del det
    torch.cuda.empty_cache()
