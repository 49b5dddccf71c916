#!/usr/bin/env python
"""DART multi-class detection throughput on B200 (BASELINE.json metric: images/sec at
1008^2 ViT-H/14 DART, N=4 and N=80 classes, on 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--classes 4] [--batch 1]
                    [--impl ours|reference] [--shard images|classes]

A step = one detection of one batch of synthetic 1008^2 scenes (SceneSpec(seed=1000+i,
num_rects=3, noise=0.05)) against N class prompts: backbone, class-batched enc-dec,
post-processing with gates open (presence 0, score 0: worst-case NMS work).  Weights are
the deterministic random init of the full ViT-H/14 model (seed 0).

The headline line (configs[1], N=4, batch 1 per GPU):
  value  = images/s over exactly K device-timed steps (CUDA events on the launch stream,
           max over ranks), inputs resident in HBM, through the inter-frame pipeline
           (Detector.detect_device_pipelined: 2 backbone streams + 1 decode stream).
  e2e    = the same through the public streaming API Detector.detect_stream() with pinned
           host images: H2D of the images, the whole path, D2H of the kept detections,
           inside the timed region.
  n80    = the same two numbers at N=80 COCO classes (configs[2]) in the same run.
  shard_classes (N>1 GPUs, or --shard classes) = config 5: 80 classes sharded over the ranks,
           backbone + enc-dec prefix of one image per rank, NCCL all-gather of the prefix
           output e1, class-shard decode of all W images, all-gather of raw outputs.
  roofline = the dominant kernel of the N=4 step (tcgen05 GEMM with the fp32 residual
           epilogue: backbone attn.out + mlp.fc2) timed live with CUDA events; roofline_attn16
           = the dominant kernel of the N=80 step (hd-16 encoder self-attention) against the
           exp (MUFU + FMA-polynomial) roof.
  cpu_baseline = the UNMODIFIED reference (baseline/_ref, pip-installed from /root/reference
           by oracle/install_ref.sh) timed per additive unit on the host cores, composed as
           the reference's own loops compose (model.py:457-458 blocks, 559-564 classes).
Multi-GPU: `--gpus N` without torchrun re-launches itself under torch.distributed.run with N
ranks (one per GPU, NCCL); image-batch data parallelism has no collective on the data path
("scaling": "weak"); timing is the max over ranks.
--impl reference: the reference CPU path alone (rank 0), same units and composition.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

METRIC = "images/sec at 1008^2 ViT-H/14 DART (N classes), B images per step"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
N80 = 80


def gflops_per_image(cfg, n_classes: int) -> float:
    """Algorithmic FLOPs (2 per MAC, reference math) with the
    class-independent prefix counted once: F(N) = F_bb + F_prefix + N * F_class."""
    T, E, L, G, H = cfg.tokens, cfg.embed_dim, cfg.num_blocks, len(cfg.global_block_indices), cfg.num_heads
    hd, w2, p, F = cfg.head_dim, cfg.window_size ** 2, cfg.patch_size, cfg.fpn_dims[0]
    nw = T // w2
    d, H2, Lt, q1, ne, nd = cfg.text_dim, cfg.num_heads, cfg.text_tokens, cfg.num_queries + 1, \
        cfg.num_encoder_layers, cfg.num_decoder_layers
    dh = d // H2
    fb = 2 * T * 3 * p * p * E + L * 24 * T * E * E + (L - G) * 4 * H * nw * w2 * w2 * hd + G * 4 * H * T * T * hd
    fb += 2 * E * F * (T + T / 4 + T / 16)
    prefix = 2 * T * F * d + 8 * T * d * d + 4 * H2 * T * T * dh + 8 * q1 * d * d + 4 * H2 * q1 * q1 * dh
    enc = ne * (4 * T * d * d + 4 * Lt * d * d + 4 * H2 * T * Lt * dh + 16 * T * d * d) + (ne - 1) * (
        8 * T * d * d + 4 * H2 * T * T * dh)
    dec = nd * (4 * q1 * d * d + 4 * T * d * d + 4 * H2 * q1 * T * dh + 16 * q1 * d * d) + (nd - 1) * (
        8 * q1 * d * d + 4 * H2 * q1 * q1 * dh)
    heads = 2 * cfg.num_queries * d * 5 + 2 * d
    return (fb + prefix + n_classes * (enc + dec + heads)) / 1e9


def load_peaks():
    try:
        with open(PEAKS_PATH) as f:
            pk = json.load(f)
        return pk, "measured"
    except Exception:
        return FALLBACK_PEAKS, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled every 10 ms through NVML while `active` (the timed
    regions only: `with sampler.timed(): ...`); nvidia-smi polling as a fallback."""

    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4,
            "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.index, self.samples, self.active, self.stop = index, [], False, False
        self.nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None
            self.max_mhz = None
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _sample(self):
        if self.nvml is not None:
            pn = self.nvml
            sm = pn.nvmlDeviceGetClockInfo(self.h, pn.NVML_CLOCK_SM)
            try:
                bits = pn.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                bits = pn.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
            return float(sm), int(bits)
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
        a = [x.strip() for x in out.split(",")]
        if self.max_mhz is None:
            self.max_mhz = float(a[1])
        return float(a[0]), 0

    def _run(self):
        while not self.stop:
            if self.active:
                try:
                    self.samples.append(self._sample())
                except Exception:
                    pass
            time.sleep(0.01)

    class _Timed:
        def __init__(self, s):
            self.s = s

        def __enter__(self):
            self.s.active = True

        def __exit__(self, *exc):
            self.s.active = False

    def timed(self):
        return ClockSampler._Timed(self)

    def summary(self):
        self.stop = True
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        sm = [s for s, _ in self.samples]
        reasons = sorted({k for _, b in self.samples for k, bit in self.BITS.items() if b & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(min(sm)), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml" if self.nvml else "nvidia-smi",
                "window": "timed regions only, 10 ms period"}


def coco80():
    return ["person", "bicycle", "car", "motorcycle", "airplane", "bus", "train", "truck", "boat", "traffic light",
            "fire hydrant", "stop sign", "parking meter", "bench", "bird", "cat", "dog", "horse", "sheep", "cow",
            "elephant", "bear", "zebra", "giraffe", "backpack", "umbrella", "handbag", "tie", "suitcase", "frisbee",
            "skis", "snowboard", "sports ball", "kite", "baseball bat", "baseball glove", "skateboard", "surfboard",
            "tennis racket", "bottle", "wine glass", "cup", "fork", "knife", "spoon", "bowl", "banana", "apple",
            "sandwich", "orange", "broccoli", "carrot", "hot dog", "pizza", "donut", "cake", "chair", "couch",
            "potted plant", "bed", "dining table", "toilet", "tv", "laptop", "mouse", "remote", "keyboard",
            "cell phone", "microwave", "oven", "toaster", "sink", "refrigerator", "book", "clock", "vase",
            "scissors", "teddy bear", "hair drier", "toothbrush"]


def class_names(n: int):
    base = ["person", "car", "dog", "bicycle"]
    if n <= 4:
        return base[:n]
    return coco80()[:n] if n <= 80 else [f"class{i:02d}" for i in range(n)]


def bench_config(args, world: int) -> dict:
    """The workload description, identical in both arms (so the driver can match them)."""
    return {"workload": f"full ViT-H/14 DART 1008^2, {args.classes} classes, batch {args.batch} per GPU",
            "classes": args.classes, "batch_per_gpu": args.batch, "secondary_classes": N80,
            "parallelism": f"image-dp{world}", "thresholds": "presence 0, score 0 (gates open)",
            "images": "SceneSpec(seed=1000+i, image_size=1008, num_rects=3, noise=0.05, num_classes=4)",
            "weights": "random init, seed 0"}


# ============================================================================ CPU reference
def _blas_threads() -> int | None:
    try:
        from threadpoolctl import threadpool_info

        return max((i.get("num_threads") or 0) for i in threadpool_info()) or None
    except Exception:
        return None


def reference_cpu_units(log=None):
    """Time the UNMODIFIED reference package (baseline/_ref; float64 NumPy, all BLAS threads)
    per additive unit of its own loops, on a model with the full-size shapes but only the
    units needed (weights are keyed by parameter path, so block 0 / block 1 / layer 0 hold
    exactly the full model's values):
        patch      = patch_tokens                        (model.py:426)
        windowed   = _block_forward(block 0, windowed)   (model.py:412)
        global     = _block_forward(block 1, global)
        fpn        = fpn_from_tokens                     (model.py:446)
        class_1x1  = _encdec_single of a 1-encoder/1-decoder-layer model, one class
                     (input proj + layer + final LN + layer + heads, model.py:511-533)
        enc_layer / dec_layer = one more layer body, the reference's own _ln/_mha/_mlp_forward
        postprocess(N) = pipeline.postprocess of N classes x 200 queries, gates open
    seconds/image(N) = patch + (L-G) windowed + G global + fpn
                       + N (class_1x1 + (ne-1) enc_layer + (nd-1) dec_layer) + postprocess(N)
    (exact for the reference: blocks and classes are independent Python loops,
    model.py:457-458, 559-564).  Falls back to the oracle port if baseline/_ref is absent."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import dart.model as M
        import dart.pipeline as PL
        from dart.scenes import SceneSpec, generate_scene
        from dart.tensors import PrecisionMode
    except ImportError:
        return None
    mode = PrecisionMode.FP32
    full = M.ModelConfig(1008, 14, 1280, 32, (7, 15, 23, 31), 24, 16, (256, 256, 256), 32, 256, 200, 6, 6, seed=0)
    unit_cfg = dataclasses.replace(full, num_blocks=2, global_block_indices=(1,), num_encoder_layers=1,
                                   num_decoder_layers=1)
    units = {}

    def timed(name, fn):
        t0 = time.perf_counter()
        r = fn()
        units[name] = time.perf_counter() - t0
        if log:
            log(f"[cpu-ref] {name}: {units[name]:.2f}s")
        return r

    t0 = time.perf_counter()
    model = M.build_model(unit_cfg, with_mask_head=False)
    build_s = time.perf_counter() - t0
    image, _ = generate_scene(SceneSpec(seed=1000, image_size=1008, num_rects=3, noise=0.05, num_classes=4))
    x = timed("patch", lambda: M.patch_tokens(model, image, mode))
    x = timed("windowed_block", lambda: M._block_forward(model, x, 0, mode))
    x = timed("global_block", lambda: M._block_forward(model, x, 1, mode))
    lv = timed("fpn", lambda: M.fpn_from_tokens(model, x, mode))
    text = M.text_encode(model, ["person"]).stack(["person"])[0]
    qf, bx, pl, sl = timed("class_1x1", lambda: M._encdec_single(model, lv[0], text, mode))
    e = M._linear(model, lv[0], "encdec.input", mode)

    def enc_layer():  # the loop body of _encdec_single (model.py:514-519)
        p = "encoder.layer0"
        h = M._ln(model, e, f"{p}.ln1")
        e2 = e + M._mha(model, h, h, f"{p}.self", mode)
        e2 = e2 + M._mha(model, M._ln(model, e2, f"{p}.ln2"), text, f"{p}.cross", mode)
        return e2 + M._mlp_forward(model, M._ln(model, e2, f"{p}.ln3"), f"{p}.mlp", mode)

    timed("enc_layer", enc_layer)
    mem = M._ln(model, e, "encoder.final_ln")

    def dec_layer():  # model.py:522-527
        q = np.concatenate([model.params["decoder.queries"], model.params["decoder.presence_token"]], axis=0)
        p = "decoder.layer0"
        h = M._ln(model, q, f"{p}.ln1")
        q = q + M._mha(model, h, h, f"{p}.self", mode)
        q = q + M._mha(model, M._ln(model, q, f"{p}.ln2"), mem, f"{p}.cross", mode)
        return q + M._mlp_forward(model, M._ln(model, q, f"{p}.ln3"), f"{p}.mlp", mode)

    timed("dec_layer", dec_layer)
    pcfg = PL.PipelineConfig(presence_threshold=0.0, score_threshold=0.0)
    for n in (4, N80):
        raw = M.RawQueryOutputs(query_features=np.stack([qf] * n), boxes=np.stack([bx] * n),
                                presence_logits=np.array([pl] * n, dtype=np.float64), score_logits=np.stack([sl] * n))
        timed(f"postprocess_n{n}", lambda: PL.postprocess(raw, class_names(n), pcfg))
    L, G = full.num_blocks, len(full.global_block_indices)
    per_class = units["class_1x1"] + (full.num_encoder_layers - 1) * units["enc_layer"] + \
        (full.num_decoder_layers - 1) * units["dec_layer"]
    shared = units["patch"] + (L - G) * units["windowed_block"] + G * units["global_block"] + units["fpn"]

    def per_image(n):
        pp = units.get(f"postprocess_n{n}", units["postprocess_n4"] * n / 4)
        return shared + n * per_class + pp

    sample = ("unmodified reference dart 0.1.0 (baseline/_ref), float64 NumPy/OpenBLAS, timed once per unit at "
              "full size on image SceneSpec(seed=1000): patch_tokens, 1 windowed + 1 global _block_forward, "
              "fpn_from_tokens, one class through _encdec_single of a 1+1-layer model, one more encoder and decoder "
              "layer, postprocess; extrapolated additively to (L-G)=28 windowed + G=4 global blocks and "
              "N x (6 enc + 6 dec) layers, exactly as the reference's loops compose")
    return {"per_image": per_image, "units_s": units, "sample": sample, "kind": "reference",
            "build_s": build_s, "cpu_s": sum(units.values())}


def oracle_port_units(log=None):
    """Fallback when baseline/_ref is missing: the float64 NumPy oracle port, same units."""
    from oracle import dart_oracle as O

    ocfg = O.full_config()
    units = {}

    def timed(name, fn):
        t0 = time.perf_counter()
        r = fn()
        units[name] = time.perf_counter() - t0
        if log:
            log(f"[cpu-port] {name}: {units[name]:.2f}s")
        return r

    decl = {p: (s, i) for p, s, i in O.param_declaration(ocfg)}
    P = {}

    def need(prefix):
        for p, (s, i) in decl.items():
            if p.startswith(prefix) and p not in P:
                if i == "ones":
                    P[p] = np.ones(s)
                elif i == "zeros":
                    P[p] = np.zeros(s)
                elif i in ("rope_cos", "rope_sin"):
                    P["rope.cos"], P["rope.sin"] = O.rope_tables(ocfg)
                else:
                    P[p] = O.philox_uniform(0, p, s, int(i))

    for pre in ("rope", "patch_embed", "backbone.block0.", "backbone.block7.", "fpn.", "encdec.", "encoder.",
                "decoder.", "text.", "heads."):
        need(pre)
    image, _ = O.scene(1000, 1008, num_classes=4)
    x = timed("patch", lambda: O.linear(P, O.patchify(ocfg, image), "patch_embed"))
    timed("windowed_block", lambda: O.backbone_block(P, ocfg, x, 0))
    timed("global_block", lambda: O.backbone_block(P, ocfg, x, 7))
    l0 = timed("fpn", lambda: O.fpn(P, ocfg, x))[0]
    text = O.text_embedding(P, ocfg, "person")
    timed("class_6x6", lambda: O.encdec_one(P, ocfg, l0, text))
    L, G = ocfg.num_blocks, len(ocfg.global_block_indices)
    shared = units["patch"] + (L - G) * units["windowed_block"] + G * units["global_block"] + units["fpn"]
    return {"per_image": lambda n: shared + n * units["class_6x6"], "units_s": units, "kind": "port",
            "sample": "oracle port (float64 NumPy) per unit at full size, composed additively", "build_s": 0.0,
            "cpu_s": sum(units.values())}


def cpu_units(log=None):
    return reference_cpu_units(log) or oracle_port_units(log)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    t0 = time.perf_counter()
    cu = cpu_units(log=lambda s: print(s, file=sys.stderr, flush=True))
    per = cu["per_image"](args.classes)
    value = 1.0 / per
    cores = os.cpu_count()
    cpu = {"value": value, "unit": "images/s", "cores": cores, "blas_threads": _blas_threads(), "kind": cu["kind"],
           "sample": cu["sample"], "units_s": cu["units_s"], "value_n80": 1.0 / cu["per_image"](N80),
           "extrapolated": True, "units_measured_once": True}
    line = {
        "impl": "reference", "metric": metric_name(args), "value": value, "unit": "images/s", "n_gpus": world,
        "steps": 1, "steps_requested": args.steps, "warmup": 0,
        "steps_note": "each additive unit of the reference's loops ran once (one step = one bounded sample); "
                      "value = 1 / (sum of units composed to one full image)",
        "ms_per_step": per * 1000.0, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (SceneSpec seed 1000, random-init ViT-H/14 weights seed 0)",
        "config": bench_config(args, world), "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "n80": {"value": cpu["value_n80"], "unit": "images/s"},
        "wall_s": time.perf_counter() - t0, "cpu_s_measured": cu["cpu_s"], "build_s": cu["build_s"],
    }
    print(json.dumps(line), flush=True)


def metric_name(args):
    return METRIC.replace("N classes", f"N={args.classes} classes").replace(
        "B images", "1 image" if args.batch == 1 else f"{args.batch} images")


# ============================================================================ B200 arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2603_11441_b200 as D
    from paper_2603_11441_b200 import _native
    from paper_2603_11441_b200.detector import Detector

    _native.load()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench: rank {rank} needs GPU {local} but only {torch.cuda.device_count()} are visible")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
    elif args.shard == "classes":  # the class-sharded protocol on a single-rank NCCL group
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
        s.close()
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    log = (lambda s: print(s, file=sys.stderr, flush=True)) if rank == 0 else (lambda s: None)
    clocks = ClockSampler(local)

    cfg = D.vit_h_config(seed=0)
    t0 = time.perf_counter()
    model = D.build_model(cfg, with_mask_head=False)
    log(f"[bench] build_model {time.perf_counter() - t0:.1f}s")
    gates_open = D.PipelineConfig(presence_threshold=0.0, score_threshold=0.0)

    B = args.batch
    n_imgs = max(2, min(8, args.steps + args.warmup))
    pool = [np.stack([D.generate_scene(D.SceneSpec(seed=1000 + rank * 100000 + i * B + j, image_size=1008,
                                                   num_rects=3, noise=0.05, num_classes=4))[0]
                      for j in range(B)]).astype(np.float32) for i in range(n_imgs)]
    dev_pool = [torch.from_numpy(p).to(dev) for p in pool]
    host_pool = [torch.from_numpy(p).pin_memory() for p in pool]
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed_ms(fn, steps, sample_clocks=True):
        """Barrier + sync, CUDA events around exactly `steps` calls on the launch stream, barrier
        + sync; max over ranks."""
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        with clocks.timed() if sample_clocks else _null():
            e0.record(stream)
            for i in range(steps):
                fn(i)
            e1.record(stream)
            barrier()
        return max_over_ranks(e0.elapsed_time(e1))

    imgs = args.steps * B * world
    h2d = B * cfg.image_size * cfg.image_size * 3 * 4

    def measure(n_classes, serial=True, defaults=True):
        """All legs of one class count: serial, pipelined (value), default gates, e2e."""
        names = class_names(n_classes)
        t0 = time.perf_counter()
        det = Detector(model, names, gates_open, device=dev)
        log(f"[bench] N={n_classes}: detector ready {time.perf_counter() - t0:.1f}s")
        r = {}
        if serial:
            for i in range(args.warmup):
                det.detect_device(dev_pool[i % n_imgs])
            barrier()
            det.reset_launch_count()
            ms = timed_ms(lambda i: det.detect_device(dev_pool[i % n_imgs]), args.steps)
            r["value_serial"] = imgs / (ms / 1000.0)
            r["ms_per_step_serial"] = ms / args.steps
            r["gpu_launches_serial"] = det.launch_count()
        # where one serial step's device time goes (CUDA events between the stages)
        r["stage_ms"] = {k: round(v, 4) for k, v in det.stage_times(dev_pool[0], reps=3).items()}
        # inter-frame pipeline (headline value)
        for i in range(args.warmup):
            det.detect_device_pipelined(dev_pool[i % n_imgs])
        det.pipeline_join()
        barrier()
        det.pipeline_reset_launch_count()

        def pipe_step(i):
            det.detect_device_pipelined(dev_pool[i % n_imgs])
            if i == args.steps - 1:
                det.pipeline_join()

        ms = timed_ms(pipe_step, args.steps)
        r["value"] = imgs / (ms / 1000.0)
        r["ms_per_step"] = ms / args.steps
        r["gpu_launches"] = det.pipeline_launch_count()
        r["nbb"] = det._pipeline(B)["nbb"]
        p = det._pipeline(B)
        res = det.result_tensors(p["slots"][(p["t"] - 1) % p["nslot"]])
        r["kept_detections_last_step"] = int(res["kc"].sum().item())
        if defaults:  # the reference's default gates (presence 0.5, score 0.45; pipeline.py:67-100)
            det_def = Detector(model, names, D.PipelineConfig(), device=dev)
            for i in range(args.warmup):
                det_def.detect_device_pipelined(dev_pool[i % n_imgs])
            det_def.pipeline_join()
            barrier()

            def def_step(i):
                det_def.detect_device_pipelined(dev_pool[i % n_imgs])
                if i == args.steps - 1:
                    det_def.pipeline_join()

            r["value_default_thresholds"] = imgs / (timed_ms(def_step, args.steps) / 1000.0)
            del det_def
        # end to end through the public API with pinned host images: H2D of the images and D2H
        # of the kept detections inside the timed region
        for _ in det.detect_stream([host_pool[i % n_imgs] for i in range(max(1, args.warmup))]):
            pass
        barrier()
        out = [None]

        def e2e_all(_):
            for res_i in det.detect_stream([host_pool[i % n_imgs] for i in range(args.steps)]):
                out[0] = res_i[0]
            det.pipeline_join()

        e2e_ms = timed_ms(e2e_all, 1)
        r["e2e"] = {"value": imgs / (e2e_ms / 1000.0), "unit": "images/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": det.d2h_bytes(B)}
        r["detections_e2e_last"] = len(out[0])
        del det
        torch.cuda.empty_cache()
        return r

    r4 = measure(args.classes)
    log(f"[bench] N={args.classes}: {r4['value']:.2f} img/s (e2e {r4['e2e']['value']:.2f})")
    r80 = None
    if not args.no_n80 and args.classes != N80:
        r80 = measure(N80, serial=False, defaults=False)
        log(f"[bench] N={N80}: {r80['value']:.2f} img/s (e2e {r80['e2e']['value']:.2f})")

    shard = None
    if world > 1 or args.shard == "classes":
        shard = measure_class_sharded(model, dev_pool, n_imgs, args, world, rank, timed_ms, barrier, log)

    roof = gemm_roofline(cfg, dev, args, stream)
    roof16 = attn16_roofline(cfg, dev, stream)

    pk, pk_kind = load_peaks()
    gf = gflops_per_image(cfg, args.classes)
    step_tflops = gf * imgs / (r4["ms_per_step"] * args.steps / 1000.0) / 1000.0 / world
    clk = clocks.summary()
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cu = cpu_units(log=log)
            cpu = {"value": 1.0 / cu["per_image"](args.classes), "unit": "images/s", "cores": os.cpu_count(),
                   "blas_threads": _blas_threads(), "kind": cu["kind"], "sample": cu["sample"],
                   "units_s": cu["units_s"], "value_n80": 1.0 / cu["per_image"](N80), "extrapolated": True}
        line = {
            "metric": metric_name(args), "value": r4["value"], "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r4["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "fp16 operands, fp32 accumulate/residual, fp64 post-processing",
            "data": "synthetic (SceneSpec seed 1000+i, random-init ViT-H/14 weights seed 0)",
            "config": dict(bench_config(args, world), schedule=(
                f"inter-frame pipeline: {r4['nbb']} backbone streams taking images in turn + 1 decode stream "
                "(enc-dec + post-processing of image t); every image fully processed"),
                l2="working set > L2 (1.29 GB fp16 weights streamed per step; 8-image input pool)"),
            "e2e": r4["e2e"],
            "gpu_launches": r4["gpu_launches"],
            "value_serial": r4.get("value_serial"), "ms_per_step_serial": r4.get("ms_per_step_serial"),
            "gpu_launches_serial": r4.get("gpu_launches_serial"),
            "stage_ms_serial": r4.get("stage_ms"),
            "value_default_thresholds": r4.get("value_default_thresholds"),
            "kept_detections_last_step": r4["kept_detections_last_step"],
            "detections_e2e_last": r4["detections_e2e_last"],
            "n80": None if r80 is None else {
                "classes": N80, "value": r80["value"], "unit": "images/s", "ms_per_step": r80["ms_per_step"],
                "e2e": r80["e2e"], "gpu_launches": r80["gpu_launches"], "stage_ms_serial": r80.get("stage_ms"),
                "kept_detections_last_step": r80["kept_detections_last_step"],
                "step_roofline_frac": gflops_per_image(cfg, N80) * r80["value"] / world / 1000.0 /
                pk["bf16_tflops_sustained"],
                "cpu_baseline_value": None if cpu is None else cpu["value_n80"]},
            "shard_classes": shard,
            "roofline": roof,
            "roofline_attn16": roof16,
            "step_roofline": {"bound": "tensor", "gflop_per_image": gf, "achieved_tflops": step_tflops,
                              "peak_tflops": pk["bf16_tflops_sustained"], "peak_kind": f"{pk_kind} sustained",
                              "frac": step_tflops / pk["bf16_tflops_sustained"]},
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def measure_class_sharded(model, dev_pool, n_imgs, args, world, rank, timed_ms, barrier, log):
    """Config 5: 80 classes sharded over the W ranks (distributed.class_sharded_raw): each round
    every rank contributes one image (backbone + enc-dec prefix), the prefix outputs are
    all-gathered over NCCL, each rank decodes its N/W classes for all W images, the raw
    outputs are all-gathered and every rank post-processes its own image.  K rounds = K*W
    images; device-timed, no host sync inside."""
    import paper_2603_11441_b200 as D
    from paper_2603_11441_b200.distributed import ClassShardPlan, NativeEngine, class_sharded_raw

    names = class_names(N80)
    cfg = D.PipelineConfig(presence_threshold=0.0, score_threshold=0.0)
    eng = NativeEngine(model)

    def step(i):
        bx, sc, pr, _ = class_sharded_raw(eng, dev_pool[i % n_imgs], names, None)
        eng.postprocess_device(bx, sc, pr, cfg)

    for i in range(args.warmup):
        step(i)
    barrier()
    ms = timed_ms(step, args.steps)
    val = args.steps * world / (ms / 1000.0)
    log(f"[bench] class-sharded N={N80} over {world} ranks: {val:.2f} img/s")
    return {"classes": N80, "value": val, "unit": "images/s", "ms_per_round": ms / args.steps, "n_gpus": world,
            "classes_per_rank": ClassShardPlan(N80, world).width,
            "exchange": "NCCL all_gather of e1 [5184, 256] fp32 per image + raw outputs [N/W, 200, 5] fp64"}


def _time_launches(fn, stream, reps=30):
    import torch

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1000.0


def gemm_roofline(cfg, dev, args, stream):
    """Dominant kernel of the N=4 step: gemm_tc_kernel with the fp32 residual epilogue (epi 3),
    one backbone attn.out ([T,1280]x[1280,1280]) and one mlp.fc2 ([T,5120]x[5120,1280]) launch per
    block, timed on the launching stream with CUDA events at the step's shapes."""
    import torch

    from paper_2603_11441_b200 import _native

    pk, pk_kind = load_peaks()
    lib = _native.load()
    M, E = args.batch * cfg.tokens, cfg.embed_dim
    out = torch.zeros(M, E, device=dev, dtype=torch.float32)
    bias = torch.zeros(E, device=dev)
    res, res_pdl = {}, {}
    # as the backbone runs them: split-K only when DART_SPLITK (mask bits 2 / 4; off by default) asks
    mask = int(os.environ.get("DART_SPLITK", "0"))
    for name, K, bit in (("attn.out", E, 2), ("mlp.fc2", 4 * E, 4)):
        lib.dart_gemm_force_splitk(2 if mask & bit else 1)
        A = torch.randn(M, K, device=dev).half()
        W = (torch.randn(E, K, device=dev) / K ** 0.5).half()
        call = lambda A=A, W=W, K=K: _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(),
                                                                 out.data_ptr(), None, M, E, K, 3, None, None, 0, 0,
                                                                 0, stream.cuda_stream))
        # kernel boundaries as in the headline's pipeline (programmatic dependent launch off) ...
        lib.dart_set_pdl(0)
        res[name] = (2.0 * M * E * K, _time_launches(call, stream))
        # ... and as on a single stream (PDL on: each launch's prologue overlaps the previous tail)
        lib.dart_set_pdl(1)
        res_pdl[name] = (2.0 * M * E * K, _time_launches(call, stream))
        lib.dart_set_pdl(-1)
        lib.dart_gemm_force_splitk(1)
    flop = sum(f for f, _ in res.values())
    t = sum(s for _, s in res.values())
    t_pdl = sum(s for _, s in res_pdl.values())
    achieved = flop / t / 1e12
    peak = pk["bf16_tflops"]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "roofline_traffic.json")) as f:
            tj = json.load(f)
        if args.batch == 1:
            traffic = sum(tj[k]["dram_read_bytes"] + tj[k]["dram_write_bytes"] for k in ("attn.out", "mlp.fc2")) / 2
    except Exception:
        pass
    return {"kernel": "gemm_tc_kernel, fp32 residual epilogue (backbone attn.out + mlp.fc2; 1 of each per block)"
                      + (", split-K" if mask & 6 else ""),
            "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "peak_kind": f"{pk_kind} burst bf16/fp16 dense",
            "flop_per_launch": flop / 2, "us_per_launch": t / 2 * 1e6,
            "per_shape": {k: {"flop": f, "us": s * 1e6, "tflops": f / s / 1e12} for k, (f, s) in res.items()},
            "launches": "back to back on one stream, programmatic dependent launch off (as in the pipeline)",
            "frac_with_pdl": flop / t_pdl / 1e12 / peak,
            "traffic": traffic,
            "traffic_note": "mean dram read+write bytes per launch of the two shapes, ncu --set full "
                            "(profiles/r02/roofline_traffic.json)"}


def attn16_roofline(cfg, dev, stream):
    """Dominant kernel of the N=80 step: hd-16 encoder self-attention over 80 classes x 16 heads x
    5184^2 scores (tcgen05 fa_tc_kernel<16>), timed on its launching stream.  Bound: exponentials
    (one per score); roof = MUFU ex2 16/clk/SM with the FMA-pipe polynomial share of the kernel
    (6 of 16), at the sampled SM clock."""
    import torch

    from paper_2603_11441_b200 import _native

    lib = _native.load()
    H, L, hd, items = cfg.num_heads, cfg.tokens, cfg.text_dim // cfg.num_heads, N80
    qkv = (torch.randn(items * L, 3 * H * hd, device=dev) * 0.5).half()
    o = torch.empty(items * L, H * hd, device=dev, dtype=torch.float16)
    call = lambda: _native.check(lib.dart_attention_qkv(qkv.data_ptr(), o.data_ptr(), items, H, L, hd, None,
                                                        stream.cuda_stream))
    t = _time_launches(call, stream, reps=5)
    exps = float(items) * H * L * L
    flops = 4.0 * exps * hd
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    clk = 1.965e9
    mufu_roof = 16 * sms * clk  # exp/s, MUFU only
    poly_roof = mufu_roof * 16 / 10  # 6 of 16 exps on the FMA pipe
    return {"kernel": "fa_tc_kernel<16,96,...> (enc self-attention, N=80)", "bound": "exp",
            "achieved": exps / t / 1e12, "unit": "Texp/s", "peak": poly_roof / 1e12,
            "frac": exps / t / poly_roof, "frac_mufu_only_roof": exps / t / mufu_roof,
            "us_per_launch": t * 1e6, "exps_per_launch": exps, "tensor_tflops": flops / t / 1e12,
            "peak_note": "16 ex2/clk/SM x SMs x 1.965 GHz, x16/10 for the 6-of-16 polynomial share"}


def spawn_ranks(args) -> int:
    """`--gpus N` without torchrun: re-launch this script under torch.distributed.run with N
    ranks on this node (one per GPU, NCCL over NVLink)."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench: --gpus {args.gpus} requested but only {have} GPU(s) are visible", file=sys.stderr)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # keep stdout to the one JSON line
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--classes", type=int, default=4)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--shard", default="images", choices=["images", "classes"],
                    help="classes: also run the class-sharded 80-class leg (always on with >1 GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-n80", action="store_true", help="skip the N=80 section of the line")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    run_ours(args)


if __name__ == "__main__":
    main()
