#!/usr/bin/env python
"""SubNetAct engine benchmark (BASELINE.json configs 2-5 on 1..8 B200 replicas).

One step = the OFA-ResNet50 subnet sweep {min, mid, max} (config 2): for each
subnet, ``ssn_actuate`` (in-place subnet switch) + ``ssn_forward`` of one
batch of synthetic 224x224 uint8 images.  Every forward follows a subnet
switch, so the SubNetAct actuation path is inside the timed region.

  value     whole-job images/s with inputs resident in HBM (CUDA events on the
            launching stream, barrier + sync on both sides, max over ranks)
  e2e       the same workload through the C-ABI with pinned HOST buffers: each
            step's images go H2D and its logits D2H inside the timed region
  roofline  the dominant kernel (tcgen05 WeightSlice conv) in the DRIVER-TIMED
            step: conv flops per step / (ms_per_step x the conv share of the
            step's device time), against the measured burst bf16 peak
  slackfit  config 4 at every N: the reference router's SlackFit decisions for
            N replicas on a bursty trace (servesim::run via tools/_bin/
            serve_live simulate, on the B200-profiled catalog CSV); rank r
            replays worker r's dispatches on its own engine, device-timed,
            max over ranks
  families  configs 3 (OFA-MBv3, bs 16-512) and 5 (BERT seq 128) batch sweeps
  cpu_baseline / cpu_baseline_families  the CPU oracle (fp32 port, all host
            threads) on bounded samples (rank 0, N = 1 only)
  cpu_baseline_torch  the config-2 sweep on a tuned CPU path (torch/oneDNN,
            extracted subnets, bs8, all host threads), informational
  parity    image 0 of each timed subnet against the oracle (checker, untimed)

Multi-GPU: one process per GPU; ``--gpus N`` under plain python re-executes
itself under torch.distributed.run.  Each rank is an independent full-supernet
replica (weak scaling; no data-path collective — only the timing barrier and
the max-over-ranks reduce).

``--impl reference`` times the reference-side CPU implementation of the path
(the oracle port — the reference itself has no tensor operators)
on the same config/metric, rank 0 only.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "subnet images/sec per B200 and 8-GPU box vs CPU ref; actuation latency (µs)"
SUBNETS = ["min", "mid", "max"]
SERVE_LIVE = os.path.join(ROOT, "tools", "_bin", "serve_live")
CATALOG_CSV = os.path.join(ROOT, "profiles", "round2", "catalog_b200.csv")
SWEEP_BATCHES = [1, 2, 4, 8, 16, 32, 64, 128, 256]


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return dict(hbm=d["hbm_gbs"], tc=d["bf16_tflops"], tc_sust=d["bf16_tflops_sustained"],
                    src="measured (MEASURED_PEAKS.json)")
    except Exception:
        return dict(hbm=6650.0, tc=1590.0, tc_sust=1400.0,
                    src="fallback (B200_PROFILING.md)")


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []  # (time, fields)
        self.proc = None
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs a few hundred ms for its first sample, longer
            # than a short timed region: wait for it, then mark the region
            deadline = time.time() + 5.0
            while not self.rows and time.time() < deadline and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def start(self):  # the timed region begins / ends (host clock)
        self.t0 = time.time()

    def stop(self):
        self.t1 = time.time()
        # one more sample after the region ends, so a region shorter than the
        # 50 ms sampling period is bracketed by samples on both sides
        deadline = self.t1 + 0.5
        while self.proc and time.time() < deadline and not any(t >= self.t1 for t, _ in self.rows):
            time.sleep(0.01)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows, bracket = self.rows, False
        if self.t0 is not None and self.t1 is not None:
            inside = [r for t, r in self.rows if self.t0 <= t <= self.t1]
            if inside:
                rows = inside
            else:  # region shorter than the sampling period: the samples either side
                before = [r for t, r in self.rows if t < self.t0][-1:]
                after = [r for t, r in self.rows if t > self.t1][:1]
                rows, bracket = before + after, True
        else:
            rows = [r for _, r in self.rows]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for i, n in enumerate(names):
                    if r[5 + i].lower().startswith("active"):
                        reasons.add(n)
            except Exception:
                pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
               "samples": len(sm)}
        if bracket:
            out["samples_bracket_region"] = True
        return out


# ---------------------------------------------------------------------------
# CPU leg (oracle port) — used by cpu_baseline and by --impl reference only

def cpu_sample(image, n_per_subnet=1, min_seconds=0.0, max_rounds=1):
    """Time the oracle's fp32 forward on n images of each sweep subnet."""
    import paper_2312_16733_b200.supernets as S
    from oracle import oracle as O
    on = O.OracleNet(2, seed=0, classes=1000, bf16_weights=True)
    x = O.images(0, 1, n_per_subnet, image)
    imgs, t0, rounds = 0, time.perf_counter(), 0
    while True:
        for sid, name in enumerate(SUBNETS):
            on.forward(S.ofa_resnet50_preset(name), x, subnet_id=sid)
            imgs += n_per_subnet
        rounds += 1
        el = time.perf_counter() - t0
        if rounds >= max_rounds and el >= min_seconds:
            break
    return imgs, el, O.lib().oracle_max_threads()


def cpu_families(seconds=3.0):
    """CPU oracle rows for configs 1, 3 and 5 (bounded samples)."""
    import paper_2312_16733_b200 as ssn
    from oracle import oracle as O
    out = {}

    def timed(fn, units):
        n, t0 = 0, time.perf_counter()
        while True:
            fn()
            n += units
            el = time.perf_counter() - t0
            if el >= seconds:
                return n / el, n, el
    on = O.OracleNet(ssn.FAMILY_TINYCNN, seed=0, classes=10, bf16_weights=False)
    x = O.images(0, 1, 8, 32)
    cfg = ssn.default_catalog_configs()[2][2]
    v, n, el = timed(lambda: on.forward(cfg, x), 8)
    out["tinycnn_config1"] = {"value": round(v, 1), "unit": "images/s",
                              "sample": f"{n} images, sub2 (W 0.6) bs8 32x32 fp32, {el:.1f} s"}
    on = O.OracleNet(ssn.FAMILY_OFA_MBV3, seed=0, classes=1000, bf16_weights=True)
    x = O.images(0, 1, 1, 224)
    cfgs = [ssn.supernets.preset(ssn.FAMILY_OFA_MBV3, s) for s in SUBNETS]
    v, n, el = timed(lambda: [on.forward(c, x) for c in cfgs], 3)
    out["ofa_mbv3_config3"] = {"value": round(v, 1), "unit": "images/s",
                               "sample": f"{n} images over {{min,mid,max}} at 224x224, {el:.1f} s"}
    on = O.OracleNet(ssn.FAMILY_BERT, seed=0, classes=2, bf16_weights=True)
    ids = O.tokens(0, 1, 1, 128)
    cfgs = [ssn.supernets.preset(ssn.FAMILY_BERT, s) for s in SUBNETS]
    v, n, el = timed(lambda: [on.forward_tokens(c, ids) for c in cfgs], 3)
    out["bert_config5"] = {"value": round(v, 1), "unit": "sequences/s",
                           "sample": f"{n} sequences over {{min,mid,max}} at seq 128, {el:.1f} s"}
    for r in out.values():
        r.update(cores=O.lib().oracle_max_threads(), kind="port", model=cpu_model())
    return out


def cpu_torch_sweep(args):
    """Informational: the same sweep on a TUNED CPU path (torch / oneDNN,
    extracted subnets, folded SubnetNorm, channels_last, all host threads;
    tests/golden/cpu_torch.py).  The oracle stays the cpu_baseline / reference
    arm; this row says what a real CPU deployment of the workload would do."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
        import cpu_torch
        r = cpu_torch.r50_sweep(args.image, batch=8, seconds=args.cpu_seconds)
        r["model"] = cpu_model()
        return r
    except Exception as e:  # informational only; never fails the bench line
        return {"unavailable": f"{type(e).__name__}: {e}"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle import oracle as O
    O.lib()
    for _ in range(args.warmup):
        cpu_sample(args.image, 1)
    times, imgs = [], 0
    for _ in range(args.steps):
        n, el, cores = cpu_sample(args.image, 1)
        times.append(el)
        imgs += n
    total = sum(times)
    value = imgs / total
    sample = f"1 image x {{{','.join(SUBNETS)}}} per step at {args.image}x{args.image}, fp32"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": "port",
                         "sample": sample, "model": cpu_model()},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": "reference (servesim) has no tensor operators (SPEC.md:8); its CPU side of this "
                "path is the oracle port oracle/ssn_oracle.c",
    }
    print(json.dumps(line), flush=True)


def workload_config(args, world):
    return {
        "workload": f"ofa_resnet50 subnet sweep {{{','.join(SUBNETS)}}}, actuate+forward per "
                    f"batch, bs{args.batch}, {args.image}x{args.image}",
        "model": "ofa_resnet50 supernet (random init, ssn_rng.h)",
        "batch": args.batch, "image": args.image, "subnets": SUBNETS,
        "global_batch": args.batch * len(SUBNETS) * world,
        "input": "uint8 NHWC images", "parallelism": f"replicas x{world}",
        "l2": "not flushed; per-step working set (96 MB weights + >1 GB activations) >> 126 MB L2",
    }


# ---------------------------------------------------------------------------
# GPU leg

def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2312_16733_b200 as ssn
    from paper_2312_16733_b200 import profiler
    from paper_2312_16733_b200.replicas import CudaTimer, timed_region

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    peaks = load_peaks()
    B = args.batch
    desc = ssn.make_desc(ssn.FAMILY_OFA_RESNET50, ssn.DTYPE_BF16, image_size=args.image,
                         num_classes=1000, max_batch=max(B, 256), seed=0,
                         input_format=ssn.INPUT_U8_NHWC)
    eng = ssn.Engine(desc, device=local_rank)
    cfgs = [ssn.ofa_resnet50_preset(n) for n in SUBNETS]
    for sid, c in enumerate(cfgs):
        eng.register_subnet(sid, c)
    # the B200 pareto catalog (config 4) as ids CAT0.. in pareto order
    CAT0 = len(SUBNETS)
    for i, (_n, _a, c) in enumerate(profiler.b200_r50_catalog()):
        eng.register_subnet(CAT0 + i, c)
    grid = sorted(set(SWEEP_BATCHES) | {B}) if not args.quick else sorted({1, 8, 64, B})
    eng.prepare(grid)
    stream = torch.cuda.Stream(device=dev)
    sptr = stream.cuda_stream
    img_bytes = args.image * args.image * 3
    xs = [torch.randint(0, 256, (B, args.image, args.image, 3), dtype=torch.uint8, device=dev)
          for _ in range(4)]
    counts = {"kernels": 0}

    def step(i, host=None):
        for sid in range(len(SUBNETS)):
            eng.actuate(sid)
            if host is None:
                eng.forward(xs[(i + sid) % 4], B, B, None, stream=sptr)
            else:
                xh, lh = host
                eng.forward(xh[(i + sid) % len(xh)], B, B, lh[sid], stream=sptr)
            counts["kernels"] += eng.stats()["last_forward_kernels"]

    # ---- device-resident timed region
    with ClockSampler(local_rank) as clk:
        for i in range(args.warmup):  # (after the sampler's first sample: the GPU is busy again)
            step(i)
        counts["kernels"] = 0
        clk.start()
        _, ms = timed_region(step, args.steps, 0, CudaTimer(torch, stream),
                             sync=torch.cuda.synchronize)
        clk.stop()
    launches = counts["kernels"]
    imgs_per_rank = args.steps * len(SUBNETS) * B
    value = world * imgs_per_rank / (ms / 1000.0)

    # ---- e2e through the C-ABI with pinned host buffers, run as a serving
    # loop: step i+1 (its H2D images, three forwards, its D2H logits) is
    # enqueued before the host reads step i's logits, so the copy engine works
    # under the previous step's kernels instead of after a drained stream.
    # Every step's H2D and D2H and the host read of every step's logits are
    # inside the timed region; two logit buffer sets alternate by step parity.
    xh = [torch.randint(0, 256, (B, args.image, args.image, 3), dtype=torch.uint8).pin_memory()
          for _ in range(2)]
    lh = [[torch.empty((B, 1000), dtype=torch.float32).pin_memory() for _ in SUBNETS]
          for _ in range(2)]
    pend = []

    def host_read():
        ev, bufs = pend.pop(0)
        ev.synchronize()
        return float(bufs[-1][0, 0])

    def e2e_step(i):
        step(i, (xh, lh[i % 2]))
        ev = torch.cuda.Event()
        ev.record(stream)
        pend.append((ev, lh[i % 2]))
        if len(pend) > 1:
            host_read()  # step i-1's logits, while step i runs

    def e2e_sync():
        while pend:
            host_read()
        torch.cuda.synchronize()

    class DrainTimer(CudaTimer):  # the last step's host read ends the region
        def stop(self):
            while pend:
                host_read()
            return super().stop()

    _, e2e_ms = timed_region(e2e_step, args.steps, args.warmup, DrainTimer(torch, stream),
                             sync=e2e_sync)
    e2e_value = world * imgs_per_rank / (e2e_ms / 1000.0)

    # ---- config 4 at every N: SlackFit dispatch across the N replicas
    slack = None if args.no_slackfit else slackfit_replay(eng, CAT0, xs[0], stream, torch, rank,
                                                          world, args)

    if rank != 0:
        eng.close()
        return

    # ---- rank 0, untimed: sweeps, actuation, roofline, parity, families, CPU
    per_subnet = {}
    for sid, name in enumerate(SUBNETS):
        row = {}
        for b in grid:
            us = eng.profile_latency(sid, b, iters=10 if b <= 64 else 5)
            row[f"bs{b}_us"] = round(us, 1)
            row[f"bs{b}_img_s"] = round(b / (us * 1e-6), 1)
        per_subnet[name] = row
    act = measure_actuation(eng, torch, stream, xs[0])
    roof = driver_roofline(eng, desc, cfgs, B, peaks, ssn, ms / args.steps)
    parity = None if args.no_parity else parity_check(eng, cfgs, xs[0], B, stream)
    families = None if args.no_families else family_rows(ssn, peaks, local_rank, args.quick)
    cpu = cpu_fam = cpu_torch = None
    if world == 1 and not args.no_cpu:
        n, el, cores = cpu_sample(args.image, 1, min_seconds=args.cpu_seconds, max_rounds=8)
        cpu = {"value": n / el, "unit": "images/s", "cores": cores, "kind": "port",
               "model": cpu_model(),
               "sample": f"{n} images over {{{','.join(SUBNETS)}}} (1 per subnet per round) at "
                         f"{args.image}x{args.image}, fp32, {el:.1f} s"}
        cpu_fam = cpu_families(seconds=3.0)
        cpu_torch = cpu_torch_sweep(args)
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (uint8 images from torch RNG; weights from ssn_rng.h seed 0; "
                "default SubnetNorm rows)",
        "config": workload_config(args, world),
        "e2e": {"value": e2e_value, "unit": "images/s",
                "mode": "serving loop: step i+1 enqueued (H2D + forwards + D2H) before the host "
                        "reads step i's logits; every copy and read inside the timed region",
                "h2d_bytes_per_step": len(SUBNETS) * B * img_bytes,
                "d2h_bytes_per_step": len(SUBNETS) * B * 1000 * 4},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "roofline": roof.pop("headline"),
        "roofline_detail": roof,
        "actuation_us": act,
        "slackfit": slack,
        "per_subnet": per_subnet,
        "families": families,
        "cpu_baseline": cpu,
        "cpu_baseline_families": cpu_fam,
        "cpu_baseline_torch": cpu_torch,
        "parity": parity,
        "engine": {k: v for k, v in eng.stats().items()
                   if k in ("weight_bytes", "norm_table_bytes", "arena_bytes", "graphs_built")},
    }
    eng.close()
    print(json.dumps(line), flush=True)


def slackfit_replay(eng, cat0, x, stream, torch, rank, world, args):
    """Config 4: the reference router (servesim::run with SlackFit over
    `world` workers, tools/_bin/serve_live simulate) decides every dispatch of
    a bursty trace on the B200-profiled catalog; rank r replays worker r's
    dispatches back to back on its engine (actuate + forward of actual_count
    padded to profiled_batch).  Device-timed, max over ranks; every rank
    derives the same schedule from the same seed (no collective)."""
    import tempfile
    from paper_2312_16733_b200.replicas import (CudaTimer, load_dispatch_log, rank_dispatches,
                                                 replay, timed_region)
    if not (os.path.exists(SERVE_LIVE) and os.path.exists(CATALOG_CSV)):
        return {"unavailable": "tools/_bin/serve_live or the catalog CSV is missing"}
    with tempfile.TemporaryDirectory() as td:
        log = os.path.join(td, "dispatch.tsv")
        out = subprocess.run([SERVE_LIVE, "simulate", "--catalog", CATALOG_CSV, "--workers",
                              str(world), "--load", str(args.slackfit_load), "--slo-factor",
                              str(args.slackfit_slo), "--duration", str(args.slackfit_seconds),
                              "--seed", "7", "--log", log],
                             check=True, capture_output=True, text=True).stdout
        sim = json.loads(out.strip().splitlines()[-1])
        recs = rank_dispatches(load_dispatch_log(log), world, rank)

    def run(_i):
        replay(eng, recs, x, cat0, stream.cuda_stream)

    _, ms = timed_region(run, 1, 1, CudaTimer(torch, stream), sync=torch.cuda.synchronize)
    total = sim["total"]
    served = total - sim["drops"]
    subs = {}
    for r in recs:
        subs[r["subnet"]] = subs.get(r["subnet"], 0) + 1
    switches = sum(1 for a, b in zip(recs, recs[1:]) if a["subnet"] != b["subnet"])
    return {"workers": world, "trace_seconds": args.slackfit_seconds,
            "load_fraction": args.slackfit_load, "slo_factor": args.slackfit_slo,
            "lambda_qps": round(sim["lambda_qps"], 1), "queries": total,
            "dispatches": sim["dispatches"], "rank0_dispatches": len(recs),
            "rank0_subnet_switches": switches, "rank0_dispatches_per_subnet": subs,
            "sim_slo_attainment": sim["slo_attainment"],
            "sim_mean_serving_accuracy": sim["mean_serving_accuracy"],
            "replay_ms_max_over_ranks": round(ms, 3),
            "served_img_s": round(served / (ms / 1000.0), 1),
            "catalog": os.path.relpath(CATALOG_CSV, ROOT),
            "note": "served images (all ranks) / slowest rank's back-to-back replay time of its "
                    "SlackFit dispatches; catalog ids are the B200 pareto subnets"}


def parity_check(eng, cfgs, x, B, stream):
    """CHECKER, outside every timed region: image 0 of the bench's own input
    batch, run on the bench's own bs-B graph of each sweep subnet (default
    SubnetNorm rows, the ids the timed steps use), against the CPU oracle
    (bf16 activation storage emulated, and pure fp32).  The oracle is never
    the thing measured."""
    import numpy as np
    from oracle import oracle as O
    on = O.OracleNet(2, seed=0, classes=1000, bf16_weights=True)
    rel = lambda a, b: float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-12))  # noqa: E731
    xs = ((x[:1].cpu().numpy().astype(np.float32) - 128.0) / 64.0).transpose(0, 3, 1, 2).copy()
    out = {}
    for sid, name in enumerate(SUBNETS):
        logits = np.zeros((B, 1000), np.float32)
        eng.actuate(sid)
        eng.forward(x, B, B, logits, stream=stream.cuda_stream)
        stream.synchronize()
        got = logits[0]
        emu = on.forward(cfgs[sid], xs, subnet_id=sid, bf16_storage=True)[0]
        ref = on.forward(cfgs[sid], xs, subnet_id=sid)[0]
        out[name] = {"rel_vs_bf16_storage_oracle": round(rel(got, emu), 5),
                     "rel_vs_fp32_oracle": round(rel(got, ref), 5),
                     "all_rows_finite": bool(np.isfinite(logits).all()),
                     "argmax_equal": bool(got.argmax() == emu.argmax())}
    out["tolerance"] = f"rel L2 <= 2e-2 (bf16); image 0 of the timed batch on the bs{B} graph"
    out["pass"] = all(v["all_rows_finite"] and v["rel_vs_bf16_storage_oracle"] <= 2e-2 and
                      v["rel_vs_fp32_oracle"] <= 2e-2 for k, v in out.items() if k in SUBNETS)
    return out


def measure_actuation(eng, torch, stream, x):
    """Host cost of ssn_actuate, and device cost of a switch: first forward
    after switching minus a steady-state forward of the same subnet."""
    host = []
    for i in range(2000):
        eng.actuate(i % 2)
        host.append(eng.stats()["last_actuate_us"])
    sptr = stream.cuda_stream

    def timed_fwd(prev, cur, n=15):
        out = []
        for _ in range(n):
            eng.actuate(prev)
            eng.forward(x, 1, 1, None, stream=sptr)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            eng.actuate(cur)
            a.record(stream)
            eng.forward(x, 1, 1, None, stream=sptr)
            b.record(stream)
            stream.synchronize()
            out.append(a.elapsed_time(b) * 1000.0)
        return statistics.median(out)

    steady = timed_fwd(2, 2)
    switched = timed_fwd(0, 2)
    return {"host_actuate_us_median": statistics.median(host),
            "host_actuate_us_p99": sorted(host)[int(0.99 * len(host))],
            "bs1_forward_steady_us": steady, "bs1_forward_after_switch_us": switched,
            "switch_overhead_us": switched - steady}


def _net_roofline_frac(ssn, desc, cfg, B, us, peaks):
    cost = ssn.plan_cost(desc, cfg)
    roof = sum(max(p["flops"] * B / (peaks["tc"] * 1e12),
                   (p["bytes"] * B + p["weight_bytes"]) / (peaks["hbm"] * 1e9))
               for p in cost["per_op"] if p is not None)
    return round(roof / (us * 1e-6), 4)


def family_rows(ssn, peaks, device, quick=False):
    """BASELINE.json configs 3 and 5 on the same engine API (untimed region):
    OFA-MobileNetV3-w1.2 over bs 16-512 (224^2 uint8 images) and the
    width/depth-sliced BERT-base encoder at seq 128 over bs 1-256, min/mid/max
    subnets.  Latency is a CUDA-graph replay (ssn_profile_latency);
    roofline_frac = sum over ops of max(flops / tensor peak, bytes / HBM peak)
    / measured latency (burst peaks)."""
    out = {}
    specs = ((ssn.FAMILY_OFA_MBV3, "ofa_mbv3_w1.2", [256] if quick else [16, 64, 256, 512], 224,
              1000, "images/s"),
             (ssn.FAMILY_BERT, "bert_base_seq128", [64] if quick else [1, 8, 64, 256], 128, 2,
              "sequences/s"))
    for fam, name, batches, size, ncls, unit in specs:
        desc = ssn.make_desc(fam, ssn.DTYPE_BF16, image_size=size, num_classes=ncls,
                             max_batch=max(batches), seed=0, input_format=ssn.INPUT_U8_NHWC)
        eng = ssn.Engine(desc, device=device)
        cfgs = [ssn.supernets.preset(fam, n) for n in SUBNETS]
        for i, c in enumerate(cfgs):
            eng.register_subnet(i, c)
        eng.prepare(batches)
        row = {"unit": unit, "batches": batches}
        for i, n in enumerate(SUBNETS):
            row[n] = {}
            for b in batches:
                us = eng.profile_latency(i, b, iters=10)
                row[n][f"bs{b}"] = {"us": round(us, 1), "value": round(b / (us * 1e-6), 1),
                                    "roofline_frac": _net_roofline_frac(ssn, desc, cfgs[i], b, us,
                                                                        peaks)}
        eng.close()
        out[name] = row
    return out


def driver_roofline(eng, desc, cfgs, B, peaks, ssn, step_ms):
    """Roofline of the dominant kernel family (tcgen05 WeightSlice conv) in
    the DRIVER-TIMED step.  Per subnet: the conv share of its device time
    (op-by-op CUDA events, ssn_profile_ops) times its graph-replay latency
    (ssn_profile_latency) gives its conv time; the per-subnet conv times are
    scaled so that the three forwards sum to the measured ms_per_step.
    achieved = algorithmic conv flops per step / conv time per step, against
    the measured BURST bf16 peak (the step is ~4 ms of tensor work)."""
    conv_f = conv_b = 0.0
    n_conv = 0
    share_t = graph_t = 0.0
    conv_roof_t = conv_op_t = 0.0
    roof_t = meas_t = 0.0
    per = {}
    for sid, cfg in enumerate(cfgs):
        cost = ssn.plan_cost(desc, cfg)
        us = eng.profile_ops(sid, B, iters=5)
        g = eng.profile_latency(sid, B, iters=10)
        c_t = a_t = f = 0.0
        for i, p in enumerate(cost["per_op"]):
            if p is None:
                continue
            t = float(us[i]) * 1e-6
            a_t += t
            fl = p["flops"] * B
            byts = p["bytes"] * B + p["weight_bytes"]
            op_roof = max(fl / (peaks["tc"] * 1e12), byts / (peaks["hbm"] * 1e9))
            roof_t += op_roof
            meas_t += t
            if p["kind"] in (1, 5):
                c_t += t
                f += fl
                conv_b += byts
                n_conv += 1
                conv_roof_t += op_roof
                conv_op_t += t
        share = c_t / a_t
        conv_f += f
        share_t += share * g
        graph_t += g
        per[SUBNETS[sid]] = {"graph_us": round(g, 1), "conv_share": round(share, 4),
                             "conv_tflops_in_graph": round(f / (share * g * 1e-6) / 1e12, 1)}
    scale = step_ms * 1e3 / graph_t   # graph-replay sum -> the driver's step time
    conv_us = share_t * scale
    achieved = conv_f / (conv_us * 1e-6) / 1e12
    # north-star target row: WeightSlice GEMMs of the LARGEST subnet at bs >= 64
    big = {}
    for bb in (64, 256):
        if bb > desc.max_batch:
            continue
        cost = ssn.plan_cost(desc, cfgs[-1])
        us = eng.profile_ops(len(cfgs) - 1, bb, iters=5)
        f = t = 0.0
        for i, p in enumerate(cost["per_op"]):
            if p is not None and p["kind"] in (1, 5):
                f += p["flops"] * bb
                t += float(us[i]) * 1e-6
        big[f"bs{bb}"] = {"conv_tflops": round(f / t / 1e12, 1),
                          "frac_burst": round(f / t / 1e12 / peaks["tc"], 4)}
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):  # ncu DRAM bytes per conv launch, same sweep (committed capture)
        with open(tfile) as fh:
            traffic = json.load(fh).get("conv_tc", {}).get("dram_bytes_per_launch")
    head = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peaks["tc"],
            "unit": "TFLOP/s", "frac": round(achieved / peaks["tc"], 4), "traffic": traffic,
            "algorithmic_bytes_per_launch": round(conv_b / max(n_conv, 1)),
            "kernel": "conv_tc_kernel / conv_halo_kernel / conv_hp_kernel (tcgen05 WeightSlice implicit GEMM), "
                      f"all conv launches of the {{{','.join(SUBNETS)}}} sweep at bs{B}",
            "peak_source": f"{peaks['src']} bf16_tflops (burst)",
            "conv_us_per_step": round(conv_us, 1),
            "conv_share_of_step": round(conv_us / (step_ms * 1e3), 4)}
    return {
        "headline": head,
        "per_subnet": per,
        "conv_flops_per_step": conv_f,
        "graph_sum_us": round(graph_t, 1),
        "driver_step_us": round(step_ms * 1e3, 1),
        "conv_hbm_gbs_op_by_op": round(conv_b / conv_op_t / 1e9, 1),
        "max_subnet_weightslice_gemm_op_by_op": big,
        "whole_net_roofline_frac_op_by_op": round(roof_t / meas_t, 4),
        "conv_roofline_frac_own_bound_op_by_op": round(conv_roof_t / conv_op_t, 4),
        "note": "headline: conv flops per step / (ms_per_step x conv share); op_by_op rows are "
                "per-launch CUDA-event times outside the graphs (no PDL overlap)",
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--image", type=int, default=224)
    ap.add_argument("--quick", action="store_true", help="small batch grids (debugging)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-families", action="store_true",
                    help="skip the OFA-MBv3 / BERT rows (configs 3 and 5)")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle parity field")
    ap.add_argument("--no-slackfit", action="store_true", help="skip the config-4 replay")
    ap.add_argument("--slackfit-load", type=float, default=0.3,
                    help="trace rate as a fraction of N x sub0 capacity (SURVEY App. B-1)")
    ap.add_argument("--slackfit-slo", type=float, default=1.5, help="SLO = x * sub5@64 latency")
    ap.add_argument("--slackfit-seconds", type=float, default=1.0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        from paper_2312_16733_b200.replicas import relaunch_under_torchrun
        sys.exit(relaunch_under_torchrun(os.path.abspath(__file__), sys.argv[1:], args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist
        if torch.cuda.device_count() < world:
            raise SystemExit(f"--gpus {world} needs {world} visible GPUs "
                             f"(found {torch.cuda.device_count()})")
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
