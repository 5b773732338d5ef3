"""Config 4: per-batch subnet switching under a bursty trace with SlackFit
dispatch, executed on the SubNetAct engine.

Pipeline (one GPU; every replica's schedule is replayed on it in turn,
which is exact for independent replicas — DESIGN.md §1 "replicas only"):
  1. profile the 6-subnet OFA-ResNet50 catalog on the B200
     (paper_2312_16733_b200.profiler) -> catalog CSV in the reference format;
  2. generate a bursty trace with the reference's own gen_bursty
     (oracle/_ref/servesim_ref gen-trace; tracegen.hpp:159-171);
  3. run the UNMODIFIED reference simulator with SlackFit on that catalog
     (servesim_ref simulate; simcore.hpp:129) -> every dispatch decision;
  4. replay each worker's dispatches on the engine: ssn_actuate(subnet) +
     ssn_forward(actual_count, profiled_batch), timed on the device;
     real completion = max(decision time, previous completion) + measured
     latency; attainment is recomputed from the trace deadlines;
  5. actuation experiment (§8f-4): the reference simulator re-run with the
     measured switch overhead vs the 100 ms model-switching baseline.
Prints one JSON line (and writes it to --out).
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF = os.path.join(ROOT, "oracle", "_ref", "servesim_ref")


def run_ref(*args):
    return subprocess.run([REF, *map(str, args)], check=True, capture_output=True, text=True).stdout


def load_trace(path):
    deadlines = {}
    with open(path) as f:
        next(f)  # spec line
        for line in f:
            q = json.loads(line)
            deadlines[q["id"]] = q["deadline_us"]
    return deadlines


def load_log(path):
    recs = []
    with open(path) as f:
        for line in f:
            p = line.rstrip("\n").split("\t")
            recs.append(dict(start=int(p[0]), completion=int(p[1]), worker=int(p[2]), subnet=int(p[3]),
                             count=int(p[4]), batch=int(p[5]), predicted=int(p[6]),
                             actuation=int(p[7]), deadline=int(p[8]),
                             ids=[int(v) for v in p[9].split(",")] if p[9] else []))
    return recs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", default="1,8")
    ap.add_argument("--load", type=float, default=0.4, help="fraction of sum(sub0 capacity)")
    ap.add_argument("--cv2", type=float, default=4.0)
    ap.add_argument("--duration", type=float, default=4.0)
    ap.add_argument("--slo-factor", type=float, default=2.0, help="SLO = factor x sub5@64 latency")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "config4.json"))
    a = ap.parse_args()

    import torch
    import paper_2312_16733_b200 as ssn
    from paper_2312_16733_b200 import profiler

    work = os.path.dirname(a.out)
    os.makedirs(work, exist_ok=True)
    desc = ssn.make_desc(ssn.FAMILY_OFA_RESNET50, ssn.DTYPE_BF16, image_size=224, num_classes=1000,
                         max_batch=64, seed=0, input_format=ssn.INPUT_U8_NHWC)
    eng = ssn.Engine(desc)
    entries = profiler.b200_r50_catalog()
    for i, (_sid, _acc, cfg) in enumerate(entries):
        eng.register_subnet(i, cfg)
    eng.prepare(profiler.REFERENCE_BATCHES)
    rows = profiler.profile_catalog(eng, entries, desc)
    csv_path = os.path.join(work, "catalog_b200.csv")
    profiler.write_catalog_csv(rows, csv_path)
    p1, p2 = profiler.holds_p1_p2(rows)
    lat = {(r[0], r[3]): r[4] for r in rows}
    cap0 = max(b * 1e6 / lat[("sub0", b)] for b in profiler.REFERENCE_BATCHES)
    slo = int(a.slo_factor * lat[("sub5", 64)])

    x = torch.randint(0, 256, (64, 224, 224, 3), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.Stream()
    result = {"catalog_csv": os.path.relpath(csv_path, ROOT), "p1": p1, "p2": p2,
              "sub0_capacity_img_s": round(cap0, 1), "slo_us": slo,
              "catalog": {r[0]: {} for r in rows}, "runs": []}
    for r in rows:
        result["catalog"][r[0]][f"bs{r[3]}_us"] = r[4]

    # measured switch overhead: first forward after a switch minus steady
    def timed(prev, cur, b, n=15):
        out = []
        for _ in range(n):
            eng.actuate(prev)
            eng.forward(x, b, b, None, stream=stream.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            eng.actuate(cur)
            e0.record(stream)
            eng.forward(x, b, b, None, stream=stream.cuda_stream)
            e1.record(stream)
            stream.synchronize()
            out.append(e0.elapsed_time(e1) * 1000)
        return statistics.median(out)
    switch_us = max(0.0, timed(0, 5, 1) - timed(5, 5, 1))
    result["measured_switch_overhead_us"] = round(switch_us, 2)

    for nw in [int(v) for v in a.workers.split(",")]:
        lam = a.load * nw * cap0
        trace = os.path.join(work, f"trace_w{nw}.jsonl")
        run_ref("gen-trace", 0.2 * lam, 0.8 * lam, a.cv2, a.duration, slo, a.seed, trace)
        log_path = os.path.join(work, f"dispatch_w{nw}.tsv")
        rep = json.loads(run_ref("simulate", csv_path, trace, nw, 0, "slackfit", log_path))
        deadlines = load_trace(trace)
        recs = load_log(log_path)
        # ---- replay every dispatch on the engine
        meas = [0.0] * len(recs)
        order = sorted(range(len(recs)), key=lambda i: (recs[i]["worker"], recs[i]["start"]))
        CH = 256
        for c0 in range(0, len(order), CH):
            chunk = order[c0:c0 + CH]
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(chunk) + 1)]
            evs[0].record(stream)
            for j, i in enumerate(chunk):
                r = recs[i]
                eng.actuate(r["subnet"])
                eng.forward(x, r["count"], r["batch"], None, stream=stream.cuda_stream)
                evs[j + 1].record(stream)
            stream.synchronize()
            for j, i in enumerate(chunk):
                meas[i] = evs[j].elapsed_time(evs[j + 1]) * 1000.0
        hits = total = 0
        acc_sum = 0.0
        busy = [0.0] * nw
        ratios = []
        prev_end = {}
        accs = [e[1] for e in entries]
        images = 0
        for i in order:
            r = recs[i]
            start = max(r["start"], prev_end.get(r["worker"], 0))
            end = start + meas[i]
            prev_end[r["worker"]] = end
            busy[r["worker"]] += meas[i]
            ratios.append(meas[i] / r["predicted"])
            images += r["count"]
            for q in r["ids"]:
                total += 1
                if end <= deadlines[q]:
                    hits += 1
                    acc_sum += accs[r["subnet"]]
        ratios.sort()
        n_q = len(deadlines)
        switches = sum(1 for i in range(1, len(order))
                       if recs[order[i]]["worker"] == recs[order[i - 1]]["worker"] and
                       recs[order[i]]["subnet"] != recs[order[i - 1]]["subnet"])
        # ---- actuation experiment on the reference simulator
        act_meas = int(math.ceil(switch_us))
        rep_act = json.loads(run_ref("simulate", csv_path, trace, nw, act_meas, "slackfit", os.devnull))
        rep_100 = json.loads(run_ref("simulate", csv_path, trace, nw, 100000, "slackfit", os.devnull))
        result["runs"].append({
            "workers": nw, "lambda_qps": round(lam, 1), "queries": n_q, "dispatches": len(recs),
            "subnet_switches": switches,
            "sim_attainment": rep.get("slo_attainment"), "sim_accuracy": rep.get("mean_serving_accuracy"),
            "replay_attainment": hits / n_q if n_q else None,
            "replay_accuracy": acc_sum / hits if hits else None,
            "measured_over_profiled_latency": {"median": round(ratios[len(ratios) // 2], 4),
                                               "p99": round(ratios[int(0.99 * (len(ratios) - 1))], 4)},
            "served_img_s_per_busy_gpu": round(images / (sum(busy) / 1e6), 1),
            "served_img_s_wall": round(images / (a.duration), 1),
            "actuation_experiment": {
                f"attainment_at_{act_meas}us": rep_act.get("slo_attainment"),
                "attainment_at_100ms": rep_100.get("slo_attainment"),
                "accuracy_at_100ms": rep_100.get("mean_serving_accuracy")},
        })
    eng.close()
    line = json.dumps(result)
    print(line)
    with open(a.out, "w") as f:
        f.write(line + "\n")


if __name__ == "__main__":
    main()
