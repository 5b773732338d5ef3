#!/usr/bin/env python
"""SubNetAct engine benchmark (BASELINE.json config 2 on 1..8 B200 replicas).

One step = the OFA-ResNet50 subnet sweep {min, mid, max}: for each subnet,
``ssn_actuate`` (in-place subnet switch) + ``ssn_forward`` of one batch of
synthetic 224x224 images.  Every forward therefore runs right after a subnet
switch — the SubNetAct actuation path is inside the timed region.

  value   whole-job images/s with inputs resident in HBM (device time, CUDA
          events on the launching stream, max over ranks)
  e2e     same workload through the C-ABI with pinned HOST buffers: the
          step's images are copied H2D and its logits D2H inside the region
  roofline  live per-op CUDA-event timing of the dominant kernel family
          (tcgen05 WeightSlice conv) vs MEASURED_PEAKS.json
  cpu_baseline  the CPU oracle (fp32 port, all host threads) on a bounded
          sample of the same workload (rank 0, N = 1 only)

Multi-GPU: one process per GPU (torchrun), each an independent full-supernet
replica doing the same per-GPU work (weak scaling, no data-path collective;
the only collectives are the timing barrier and the max-over-ranks reduce).

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


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return dict(hbm=d["hbm_gbs"], tc=d["bf16_tflops"], tc_sust=d["bf16_tflops_sustained"],
                    src="measured")
    except Exception:
        return dict(hbm=6650.0, tc=1590.0, tc_sust=1400.0, src="fallback")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

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
        for r in self.rows:
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
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU leg (oracle port) — used by cpu_baseline and by --impl reference

def cpu_sample(image, n_per_subnet=1, min_seconds=0.0, max_rounds=1):
    """Time the oracle's fp32 forward on n images of each sweep subnet."""
    import numpy as np
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
                         "sample": sample},
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
    import numpy as np
    import torch
    import paper_2312_16733_b200 as ssn

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
    grid = sorted({1, B} | ({8, 64, 256} if args.sweep else set()))
    eng.prepare(grid)
    stream = torch.cuda.Stream(device=dev)
    sptr = stream.cuda_stream
    img_bytes = args.image * args.image * 3
    xs = [torch.randint(0, 256, (B, args.image, args.image, 3), dtype=torch.uint8, device=dev)
          for _ in range(4)]

    def step(i, host=None):
        k = 0
        for sid in range(len(SUBNETS)):
            eng.actuate(sid)
            if host is None:
                eng.forward(xs[(i + sid) % 4], B, B, None, stream=sptr)
            else:
                xh, lh = host
                eng.forward(xh[(i + sid) % len(xh)], B, B, lh[sid], stream=sptr)
            k += eng.stats()["last_forward_kernels"]
        return k

    from paper_2312_16733_b200.replicas import barrier, max_over_ranks

    # ---- device-resident timed region
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for i in range(args.steps):
            launches += step(i)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1))
    imgs_per_rank = args.steps * len(SUBNETS) * B
    value = world * imgs_per_rank / (ms / 1000.0)

    # ---- e2e through the C-ABI with pinned host buffers
    xh = [torch.randint(0, 256, (B, args.image, args.image, 3), dtype=torch.uint8).pin_memory()
          for _ in range(2)]
    lh = [torch.empty((B, 1000), dtype=torch.float32).pin_memory() for _ in SUBNETS]
    for i in range(args.warmup):
        step(i, (xh, lh))
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for i in range(args.steps):
        step(i, (xh, lh))
        stream.synchronize()  # the step's logits are read on the host
        _ = float(lh[-1][0, 0])
    f1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1))
    e2e_value = world * imgs_per_rank / (e2e_ms / 1000.0)

    if rank != 0:
        eng.close()
        return

    # ---- per-subnet latency, actuation, live roofline (untimed region)
    per_subnet = {}
    for sid, name in enumerate(SUBNETS):
        row = {}
        for b in grid:
            us = eng.profile_latency(sid, b, iters=10)
            row[f"bs{b}_us"] = round(us, 1)
            row[f"bs{b}_img_s"] = round(b / (us * 1e-6), 1)
        per_subnet[name] = row
    act = measure_actuation(eng, torch, stream, xs[0], B)

    roof = live_roofline(eng, desc, cfgs, B, peaks, ssn)
    parity = None if args.no_parity else parity_check(eng, cfgs, xs[0], B, stream, torch)
    families = None if args.no_families else family_rows(ssn, peaks, local_rank)
    cpu = None
    if world == 1 and not args.no_cpu:
        n, el, cores = cpu_sample(args.image, 1, min_seconds=args.cpu_seconds, max_rounds=8)
        cpu = {"value": n / el, "unit": "images/s", "cores": cores, "kind": "port",
               "sample": f"{n} images over {{{','.join(SUBNETS)}}} (1 per subnet per round) at "
                         f"{args.image}x{args.image}, fp32, {el:.1f} s"}
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (uint8 images from torch RNG; weights from ssn_rng.h seed 0; "
                "default SubnetNorm rows)",
        "config": workload_config(args, world),
        "e2e": {"value": e2e_value, "unit": "images/s",
                "h2d_bytes_per_step": len(SUBNETS) * B * img_bytes,
                "d2h_bytes_per_step": len(SUBNETS) * B * 1000 * 4},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "roofline": roof.pop("headline"),
        "roofline_detail": roof,
        "actuation_us": act,
        "per_subnet": per_subnet,
        "families": families,
        "cpu_baseline": cpu,
        "parity": parity,
        "engine": {k: v for k, v in eng.stats().items()
                   if k in ("weight_bytes", "norm_table_bytes", "arena_bytes", "graphs_built")},
    }
    eng.close()
    print(json.dumps(line), flush=True)


def parity_check(eng, cfgs, x, B, stream, torch):
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


def measure_actuation(eng, torch, stream, x, B):
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


def family_rows(ssn, peaks, device):
    """BASELINE.json configs 3 and 5 on the same engine API (untimed region):
    OFA-MobileNetV3-w1.2 at bs256 (224^2 uint8 images) and the width/depth-
    sliced BERT-base encoder at bs64 x seq128, min/mid/max subnets.  Latency is
    a CUDA-graph replay (ssn_profile_latency); roofline_frac = sum over ops of
    max(flops / tensor peak, bytes / HBM peak) / measured latency."""
    out = {}
    specs = ((ssn.FAMILY_OFA_MBV3, "ofa_mbv3_w1.2", 256, 224, 1000, "images/s"),
             (ssn.FAMILY_BERT, "bert_base_seq128", 64, 128, 2, "sequences/s"))
    for fam, name, B, size, ncls, unit in specs:
        desc = ssn.make_desc(fam, ssn.DTYPE_BF16, image_size=size, num_classes=ncls, max_batch=B,
                             seed=0, input_format=ssn.INPUT_U8_NHWC)
        eng = ssn.Engine(desc, device=device)
        names = ("min", "mid", "max")
        cfgs = [ssn.supernets.preset(fam, n) for n in names]
        for i, c in enumerate(cfgs):
            eng.register_subnet(i, c)
        eng.prepare([B])
        row = {"batch": B, "unit": unit}
        for i, n in enumerate(names):
            us = eng.profile_latency(i, B, iters=10)
            cost = ssn.plan_cost(desc, cfgs[i])
            roof = sum(max(p["flops"] * B / (peaks["tc_sust"] * 1e12),
                           (p["bytes"] * B + p["weight_bytes"]) / (peaks["hbm"] * 1e9))
                       for p in cost["per_op"] if p is not None)
            row[n] = {"us": round(us, 1), "value": round(B / (us * 1e-6), 1),
                      "roofline_frac": round(roof / (us * 1e-6), 4)}
        eng.close()
        out[name] = row
    return out


def live_roofline(eng, desc, cfgs, B, peaks, ssn):
    """Per-op CUDA-event times of each sweep subnet at batch B; the dominant
    kernel family is the tcgen05 WeightSlice conv (OP_CONV / OP_LINEAR)."""
    tot_f = tot_t = tot_b = 0.0
    roof_t = meas_t = 0.0
    conv_t = all_t = 0.0
    conv_roof_t = 0.0
    n_conv = 0
    largest = None
    for sid, cfg in enumerate(cfgs):
        cost = ssn.plan_cost(desc, cfg)
        us = eng.profile_ops(sid, B, iters=5)
        for i, p in enumerate(cost["per_op"]):
            if p is None:
                continue
            r = p
            t = float(us[i]) * 1e-6
            all_t += t
            f = p["flops"] * B
            byts = p["bytes"] * B + p["weight_bytes"]
            op_roof = max(f / (peaks["tc_sust"] * 1e12), byts / (peaks["hbm"] * 1e9))
            roof_t += op_roof
            meas_t += t
            if r["kind"] in (1, 5):
                n_conv += 1
                conv_t += t
                conv_roof_t += op_roof
                tot_f += f
                tot_b += byts
                tot_t += t
                if sid == len(cfgs) - 1:
                    largest = largest or {"f": 0.0, "t": 0.0}
                    largest["f"] += f
                    largest["t"] += t
    achieved = tot_f / tot_t / 1e12
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
                          "frac": round(f / t / 1e12 / peaks["tc_sust"], 4)}
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):  # ncu DRAM bytes per conv_tc launch, same sweep (committed capture)
        with open(tfile) as f:
            traffic = json.load(f).get("conv_tc", {}).get("dram_bytes_per_launch")
    head = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peaks["tc_sust"],
            "unit": "TFLOP/s", "frac": round(achieved / peaks["tc_sust"], 4), "traffic": traffic,
            "algorithmic_bytes_per_launch": round(tot_b / max(n_conv, 1)),
            "kernel": "conv_tc_kernel (tcgen05 WeightSlice implicit GEMM), all launches of the "
                      f"{{{','.join(SUBNETS)}}} sweep at bs{B}",
            "peak_source": f"{peaks['src']} bf16_tflops_sustained"}
    return {
        "headline": head,
        "conv_share_of_gpu_time": round(conv_t / all_t, 4),
        "conv_hbm_gbs": round(tot_b / tot_t / 1e9, 1),
        "conv_hbm_frac": round(tot_b / tot_t / 1e9 / peaks["hbm"], 4),
        "max_subnet_conv_tflops": round(largest["f"] / largest["t"] / 1e12, 1) if largest else None,
        "max_subnet_weightslice_gemm": big,
        "whole_net_roofline_frac": round(roof_t / meas_t, 4),
        # each conv launch against ITS bound (tensor or HBM), summed over the sweep
        "conv_roofline_frac_own_bound": round(conv_roof_t / conv_t, 4),
        "note": "achieved = algorithmic 2*MAC of active WeightSlice extents / summed per-launch "
                "CUDA-event time; whole_net = sum_op max(flops/tc, bytes/hbm) / sum_op measured",
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--image", type=int, default=224)
    ap.add_argument("--sweep", action="store_true", help="also profile bs 1/8/64/256")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-families", action="store_true",
                    help="skip the OFA-MBv3 / BERT rows (configs 3 and 5)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle parity field")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist
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
