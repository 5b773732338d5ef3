// ref_driver.cpp — TEST INFRASTRUCTURE. A thin CLI over the UNMODIFIED
// reference scheduling path (servesim headers under /root/reference, compiled
// by oracle/Makefile into oracle/_ref/servesim_ref).  It is the
// subnet-selection oracle: the engine keeps the reference's SlackFit as its
// caller (no mirror of it exists here), and the tests pin that caller's
// decisions and dispatch logs to the frozen values of the reference's own
// tests.  No reference source is copied into this repo.
//
//   servesim_ref decide   <catalog.csv|default> <bucket_count> <slack_us>...
//       one line per slack: "<slack> <batch> <subnet_index> <latency_us>"
//       or "<slack> drop"        (policy.hpp:191-214, decide_slackfit 120-150)
//   servesim_ref gen-trace <base_rate> <variant_rate> <cv2> <duration_s>
//                          <slo_us> <seed> <out.jsonl>    (tracegen.hpp:159)
//   servesim_ref simulate <catalog.csv|default> <trace.jsonl> <workers>
//                          <actuation_us> <policy> <log.tsv>
//       runs servesim::run (simcore.hpp:129) with a DispatchLog; writes one
//       TSV row per dispatch and prints the report JSON (metrics.hpp:108).
#include <fstream>
#include <iostream>
#include <string>

#include "servesim/metrics.hpp"
#include "servesim/policy.hpp"
#include "servesim/profile.hpp"
#include "servesim/simcore.hpp"
#include "servesim/tracegen.hpp"

using namespace servesim;

static Catalog load(const std::string& arg) {
  if (arg == "default") return default_catalog();
  Catalog c = load_catalog(arg);
  return pareto_filter(c);
}

int main(int argc, char** argv) try {
  if (argc < 2) {
    std::cerr << "usage: servesim_ref decide|gen-trace|simulate ...\n";
    return 2;
  }
  const std::string cmd = argv[1];
  if (cmd == "decide" && argc >= 4) {
    const Catalog cat = load(argv[2]);
    const BucketTable buckets = build_buckets(cat, std::stoul(argv[3]));
    for (int i = 4; i < argc; ++i) {
      const SlackMicros slack = std::stoll(argv[i]);
      const auto d = decide(PolicyKind::slackfit(), slack, 64, buckets, cat);
      if (d)
        std::cout << slack << ' ' << d->batch_size << ' ' << d->subnet_index
                  << ' ' << d->predicted_latency_us << '\n';
      else
        std::cout << slack << " drop\n";
    }
    return 0;
  }
  if (cmd == "gen-trace" && argc == 9) {
    TraceSpec spec;
    spec.kind = TraceKind::Bursty;
    spec.base_rate = std::stod(argv[2]);
    spec.variant_rate = std::stod(argv[3]);
    spec.cv2 = std::stod(argv[4]);
    spec.duration_s = std::stod(argv[5]);
    spec.slo_us = std::stoull(argv[6]);
    spec.seed = std::stoull(argv[7]);
    save_trace(generate_trace(spec), argv[8]);
    return 0;
  }
  if (cmd == "simulate" && argc == 8) {
    const Catalog cat = load(argv[2]);
    const Trace trace = load_trace(argv[3]);
    SimConfig cfg;
    cfg.worker_count = static_cast<std::uint32_t>(std::stoul(argv[4]));
    cfg.actuation_delay_us = std::stoull(argv[5]);
    cfg.policy = policy_from_string(argv[6]);
    DispatchLog log;
    const SimReport rep = run(trace, cat, cfg, &log);
    std::ofstream out(argv[7]);
    for (const auto& r : log) {
      out << r.start_us << '\t' << r.completion_us << '\t' << r.worker << '\t'
          << r.subnet_index << '\t' << r.actual_count << '\t'
          << r.profiled_batch << '\t' << r.predicted_latency_us << '\t'
          << r.actuation_us << '\t' << r.batch_deadline_us << '\t';
      for (std::size_t i = 0; i < r.query_ids.size(); ++i)
        out << (i ? "," : "") << r.query_ids[i];
      out << '\n';
    }
    std::cout << report_to_json(rep).dump() << '\n';
    return 0;
  }
  std::cerr << "bad arguments\n";
  return 2;
} catch (const std::exception& e) {
  std::cerr << "error: " << e.what() << '\n';
  return 2;
}
