// serve_live.cpp — §8f of SURVEY.md on real engines, in C++ against the
// UNMODIFIED reference headers (servesim, /root/reference/proj/include).
//
//   profile   Supernet profiler: l_phi(B) of the six
//             OFA-ResNet50 pareto subnets measured on the engine
//             (ssn_profile_latency), written with the reference's own
//             write_catalog_csv (profile.hpp:446-461) and read back through
//             parse_catalog_csv (profile.hpp:392-444, P1 enforced) + P2 check
//             (profile.hpp:211-227).                                  (§8f-1)
//   serve     servesim's live mode with engine-backed workers
//             (include/ssn_serve.hpp; the sleep of serve_runtime.hpp:167
//             replaced by ssn_actuate + ssn_forward), next to the reference
//             simulator `run` (simcore.hpp:129) on the same bursty trace
//             (gen_bursty, tracegen.hpp:159-171) — the acceptance.cpp:429-452
//             criterion-12 analog (|d attainment| <= 0.02, |d accuracy| <=
//             0.5).                                                   (§8f-2)
//   memory    MemorySpec filled with the engine's measured bytes and run
//             through the reference memory_footprint (profile.hpp:512-545):
//             re-tests PAPER.md:451 (2.6x) and :406/485 (500x).       (§8f-3)
//   actuation the reference simulator with the MEASURED actuation cost vs the
//             100 ms model-switching baseline (simcore.hpp:247-252,
//             acceptance.cpp:271-285).                                (§8f-4)
//   simulate  the reference router's SlackFit dispatch log for N replicas
//             (servesim::run), replayed per rank by bench.py.      (config 4)
//
// Every mode prints one JSON object.  Payloads: `Query` carries no image
// (edf_queue.hpp:16-31); a batch's images are a contiguous slice of a
// device-resident pool of synthetic uint8 224x224 images (ssn_rng.h), picked
// by the batch's first query id.
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <random>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "servesim/metrics.hpp"
#include "servesim/policy.hpp"
#include "servesim/profile.hpp"
#include "servesim/serve_runtime.hpp"
#include "servesim/simcore.hpp"
#include "servesim/tracegen.hpp"
#include "ssn.hpp"
#include "ssn_rng.h"
#include "ssn_serve.hpp"

using nlohmann::json;
using servesim::Micros;

namespace {

// ---- the B200 OFA-ResNet50 catalog (paper_2312_16733_b200/profiler.py
// B200_R50_CATALOG): six uniform (d, e-index, w-index) subnets whose MACs
// mirror the reference default catalog (profile.hpp:477-486), with the
// reference's accuracies.
const double kWidths[3] = {0.65, 0.8, 1.0};
const double kExpands[3] = {0.2, 0.25, 0.35};
struct CatRow {
  const char* id;
  double acc;
  int d, e, w;
};
const CatRow kCatalog[6] = {{"sub0", 73.82, 0, 0, 0}, {"sub1", 76.69, 1, 1, 0},
                            {"sub2", 77.64, 1, 2, 0}, {"sub3", 78.25, 1, 1, 2},
                            {"sub4", 79.44, 1, 2, 2}, {"sub5", 80.16, 2, 2, 2}};

// OFA (d, e, w) -> engine control tuple (supernets.py
// ofa_resnet50_config): D = [stem_res, s1b2, s1b3, ..., s4b3].
servesim::SubnetConfig ofa_r50(int d, int e, int w) {
  servesim::SubnetConfig c;
  c.depth_flags = {d == 2};
  for (int s = 0; s < 4; ++s) {
    c.depth_flags.push_back(d >= 1);
    c.depth_flags.push_back(d >= 2);
  }
  c.expand_ratios.assign(18, kExpands[e]);
  c.width_multipliers.assign(6, kWidths[w]);
  return c;
}

ssn_supernet_desc r50_desc(uint32_t max_batch) {
  ssn_supernet_desc d{};
  d.family = SSN_FAMILY_OFA_RESNET50;
  d.dtype = SSN_DTYPE_BF16;
  d.image_size = 224;
  d.num_classes = 1000;
  d.max_batch = max_batch;
  d.input_format = SSN_INPUT_U8_NHWC;
  d.seed = 0;
  return d;
}

std::map<std::string, std::string> parse_args(int argc, char** argv, int first) {
  std::map<std::string, std::string> a;
  for (int i = first; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) throw std::invalid_argument("bad argument " + k);
    a[k.substr(2)] = (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) ? argv[++i] : "1";
  }
  return a;
}

std::string arg(const std::map<std::string, std::string>& a, const char* k, const char* def) {
  auto it = a.find(k);
  return it == a.end() ? def : it->second;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr size_t kImg = 224 * 224 * 3;
constexpr uint32_t kPool = 256;

// Synthetic payload image #i of the pool: ssn_rng.h stream kind 5 (image
// batch ordinal 900), uint8 = floor(u01 * 256).
std::vector<uint8_t> make_pool() {
  std::vector<uint8_t> h(kPool * kImg);
  for (size_t i = 0; i < h.size(); ++i)
    h[i] = static_cast<uint8_t>(ssn_u01(0, ssn_stream(SSN_STREAM_IMAGE, 900), i) * 256.0f);
  return h;
}

// Registers the catalog on `eng` (pareto order = subnet_index) with the
// catalog's control tuples, builds the graph grid.
void register_catalog(ssn::Engine& eng, const servesim::Catalog& cat) { eng.register_catalog(cat); }

servesim::Catalog with_configs(servesim::Catalog cat) {
  for (auto& rec : cat.subnets) {
    bool found = false;
    for (const auto& r : kCatalog)
      if (rec.id == r.id) {
        rec.config = ofa_r50(r.d, r.e, r.w);
        found = true;
      }
    if (!found) throw std::invalid_argument("catalog subnet " + rec.id + " has no control tuple");
  }
  return cat;
}

// Host ssn_actuate cost and the device switch overhead (first bs1 forward
// after a switch minus a steady one), on engine `eng` (catalog registered).
json measure_actuation(ssn::Engine& eng, const void* x) {
  std::vector<double> host;
  for (int i = 0; i < 2000; ++i) {
    eng.actuate(i % 2);
    host.push_back(eng.stats().last_actuate_us);
  }
  auto timed = [&](uint32_t prev, uint32_t cur) {
    std::vector<double> v;
    for (int i = 0; i < 21; ++i) {
      eng.actuate(prev);
      eng.forward(x, 1, 1, nullptr);
      eng.synchronize();
      eng.actuate(cur);
      const auto t0 = std::chrono::steady_clock::now();
      eng.forward(x, 1, 1, nullptr);
      eng.synchronize();
      v.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    }
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  const double steady = timed(5, 5), switched = timed(0, 5);
  std::sort(host.begin(), host.end());
  return {{"host_actuate_us_median", host[host.size() / 2]},
          {"host_actuate_us_p99", host[host.size() * 99 / 100]},
          {"bs1_forward_steady_us", steady},
          {"bs1_forward_after_switch_us", switched},
          {"switch_overhead_us", std::max(0.0, switched - steady)}};
}

// ---------------------------------------------------------------- profile
int cmd_profile(const std::map<std::string, std::string>& a) {
  const std::string out = arg(a, "out", "catalog_b200.csv");
  const int iters = std::stoi(arg(a, "iters", "20"));
  const double margin = std::stod(arg(a, "margin", "1.03"));
  std::vector<uint32_t> grid;
  {
    std::stringstream ss(arg(a, "batches", "1,2,4,8,16,32,64"));
    for (std::string t; std::getline(ss, t, ',');) grid.push_back(std::stoul(t));
  }
  const int nsub = std::stoi(arg(a, "subnets", "6"));
  ssn::Engine eng(std::stoi(arg(a, "device", "0")), r50_desc(grid.back()));
  servesim::Catalog cat;
  cat.max_batch = grid.back();
  for (int i = 0; i < nsub; ++i) {
    servesim::SubnetRecord rec;
    rec.id = kCatalog[i].id;
    rec.accuracy = kCatalog[i].acc;
    rec.config = ofa_r50(kCatalog[i].d, kCatalog[i].e, kCatalog[i].w);
    eng.register_subnet(static_cast<uint32_t>(i), rec.config);
    cat.subnets.push_back(rec);
  }
  eng.prepare(grid);
  json prov = json::array();
  for (int i = 0; i < nsub; ++i) {
    // MACs of the active slices (ssn_plan_ops)
    ssn::CfgView v(cat.subnets[i].config);
    ssn_supernet_desc d = r50_desc(grid.back());
    std::vector<ssn_op_info> ops(512);
    uint32_t n = 0;
    ssn::check(ssn_plan_ops(&d, &v.c, ops.data(), 512, &n));
    double macs = 0;
    for (uint32_t k = 0; k < n; ++k) {
      const auto& o = ops[k];
      if (!o.active || (o.kind != 1 && o.kind != 5)) continue;
      const double kk = static_cast<double>(o.k) * o.k;
      macs += static_cast<double>(o.hout) * o.wout * o.cout * (o.depthwise ? kk : kk * o.cin);
    }
    cat.subnets[i].gflops = std::round(macs / 1e9 * 1000) / 1000;
    Micros prev = 0;
    for (uint32_t b : grid) {
      const double med = eng.profile_latency_us(static_cast<uint32_t>(i), b, iters);
      // conservative like ceil_entry (profile.hpp:92-98); P1 tie broken by +1 us
      Micros us = static_cast<Micros>(std::ceil(margin * med));
      const bool tie = us <= prev;
      if (tie) us = prev + 1;
      prev = us;
      cat.subnets[i].profile.push_back({b, us});
      prov.push_back({{"subnet", kCatalog[i].id}, {"batch", b}, {"median_us", med}, {"latency_us", us},
                      {"p1_tiebreak", tie}});
    }
  }
  {
    std::ofstream f(out);
    servesim::write_catalog_csv(cat, f);
  }
  // read back through the reference parser: P1 is enforced there
  const servesim::Catalog back = servesim::load_catalog(out);
  std::string why;
  const bool p2 = servesim::holds_p2(back, &why);
  const servesim::Catalog par = servesim::pareto_filter(back);
  json j{{"mode", "profile"}, {"csv", out}, {"subnets", back.size()}, {"batches", grid},
         {"p1", true}, {"p2", p2}, {"p2_note", why}, {"pareto_size", par.size()},
         {"margin", margin}, {"iters", iters}, {"rows", prov}};
  std::cout << j.dump() << std::endl;
  return 0;
}

// ---------------------------------------------------------------- serve
int cmd_serve(const std::map<std::string, std::string>& a) {
  const servesim::Catalog cat = with_configs(servesim::pareto_filter(
      servesim::load_catalog(arg(a, "catalog", "catalog_b200.csv"))));
  const uint32_t workers = std::stoul(arg(a, "workers", "1"));
  int ndev = 0;
  cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  const double load = std::stod(arg(a, "load", "0.3"));
  const double cv2 = std::stod(arg(a, "cv2", "4"));
  const double duration = std::stod(arg(a, "duration", "5"));
  const double slo_factor = std::stod(arg(a, "slo-factor", "3"));
  std::vector<uint64_t> seeds;
  {
    std::stringstream ss(arg(a, "seeds", "21,22,23"));
    for (std::string t; std::getline(ss, t, ',');) seeds.push_back(std::stoull(t));
  }
  const std::string dump = arg(a, "dump-first", "");

  // engines: worker i on device i % ndev (one per GPU when workers <= GPUs)
  std::vector<std::unique_ptr<ssn::Engine>> engines;
  std::vector<ssn::Engine*> eptr;
  std::vector<uint8_t*> pools(ndev, nullptr);
  const std::vector<uint8_t> host_pool = make_pool();
  for (uint32_t i = 0; i < workers; ++i) {
    const int dev = static_cast<int>(i % ndev);
    engines.push_back(std::make_unique<ssn::Engine>(dev, r50_desc(cat.max_batch)));
    register_catalog(*engines.back(), cat);
    eptr.push_back(engines.back().get());
    if (!pools[dev]) {
      cuda_check(cudaSetDevice(dev), "cudaSetDevice");
      cuda_check(cudaMalloc(&pools[dev], host_pool.size()), "cudaMalloc pool");
      cuda_check(cudaMemcpy(pools[dev], host_pool.data(), host_pool.size(), cudaMemcpyHostToDevice), "pool upload");
    }
  }
  const json act = measure_actuation(*engines[0], pools[0]);
  const Micros act_us = static_cast<Micros>(std::ceil(act["switch_overhead_us"].get<double>() +
                                                      act["host_actuate_us_median"].get<double>()));
  auto offset = [&](const servesim::Batch& b) {
    return static_cast<size_t>(b.queries.front().id % (kPool - cat.max_batch + 1));
  };
  std::atomic<bool> dumped{false};
  std::vector<float> dump_logits(static_cast<size_t>(cat.max_batch) * 1000);
  struct DumpInfo {
    size_t off = 0;
    uint32_t count = 0;
    std::size_t subnet = 0;
  } dinfo;
  ssn::Payload payload;
  payload.images = [&](const servesim::Batch& b, uint32_t w, std::size_t) -> const void* {
    return pools[w % ndev] + offset(b) * kImg;
  };
  payload.logits = [&](const servesim::Batch& b, uint32_t w, std::size_t subnet) -> float* {
    if (dump.empty() || w != 0 || dumped.exchange(true)) return nullptr;
    dinfo.off = offset(b);
    dinfo.count = b.size();
    dinfo.subnet = subnet;
    return dump_logits.data();
  };

  // capacity of sub0 (the reference's sustainable_qps definition, simcore.hpp:73-83)
  const double cap0 = servesim::sustainable_qps(cat, cat.at(0).id, 1);
  const Micros slo = static_cast<Micros>(slo_factor * cat.at(cat.size() - 1).max_latency());
  json runs = json::array();
  bool ok = true;
  for (uint64_t seed : seeds) {
    servesim::TraceSpec spec;
    spec.kind = servesim::TraceKind::Bursty;
    const double lam = load * workers * cap0;  // stay below SlackFit's collapse
    spec.base_rate = 0.2 * lam;
    spec.variant_rate = 0.8 * lam;
    spec.cv2 = cv2;
    spec.duration_s = duration;
    spec.slo_us = slo;
    spec.seed = seed;
    const servesim::Trace trace = servesim::generate_trace(spec);
    servesim::ServeConfig lc;
    lc.worker_count = workers;
    lc.actuation_delay_us = act_us;
    lc.policy = servesim::PolicyKind::slackfit();
    servesim::DispatchLog llog;
    const ssn::LiveResult live = ssn::serve_engines(trace, cat, lc, eptr, payload, &llog);
    servesim::SimConfig sc;
    sc.worker_count = workers;
    sc.actuation_delay_us = act_us;
    sc.policy = servesim::PolicyKind::slackfit();
    const servesim::SimReport sim = servesim::run(trace, cat, sc);
    const double datt = std::abs(live.report.aggregates.slo_attainment - sim.aggregates.slo_attainment);
    const double dacc = std::abs(live.report.aggregates.mean_serving_accuracy.value_or(0.0) -
                                 sim.aggregates.mean_serving_accuracy.value_or(0.0));
    std::vector<double> ratio;
    uint64_t images = 0, switches = 0;
    double busy_us = 0;
    for (const auto& d : live.dispatches) {
      ratio.push_back(static_cast<double>(d.completion_us - d.start_us) / static_cast<double>(d.predicted_us));
      images += d.count;
      switches += d.switched;
      busy_us += static_cast<double>(d.completion_us - d.start_us);
    }
    std::sort(ratio.begin(), ratio.end());
    const bool pass = datt <= 0.02 && dacc <= 0.5 && !live.report.pacing_overrun;
    ok = ok && pass;
    runs.push_back({{"seed", seed},
                    {"lambda_qps", lam},
                    {"queries", trace.queries.size()},
                    {"live", servesim::report_to_json(live.report)},
                    {"sim", servesim::report_to_json(sim)},
                    {"d_attainment", datt},
                    {"d_accuracy", dacc},
                    {"criterion12_pass", pass},
                    {"dispatches", live.dispatches.size()},
                    {"subnet_switches", switches},
                    {"served_images", images},
                    {"served_img_s_wall", images / live.wall_s},
                    {"served_img_s_busy", images / (busy_us / 1e6)},
                    {"wall_s", live.wall_s},
                    {"service_over_profiled", {{"median", ratio.empty() ? 0 : ratio[ratio.size() / 2]},
                                               {"p99", ratio.empty() ? 0 : ratio[ratio.size() * 99 / 100]}}}});
  }
  if (!dump.empty() && dumped) {
    // the first dispatch of worker 0: header {pool offset, count, subnet},
    // its images (uint8 NHWC), its logits (float32 [count][1000])
    std::ofstream f(dump, std::ios::binary);
    uint32_t row = 0;  // the dispatched subnet's row of kCatalog (its control tuple)
    for (uint32_t r = 0; r < 6; ++r)
      if (cat.at(dinfo.subnet).id == kCatalog[r].id) row = r;
    const uint32_t hdr[4] = {static_cast<uint32_t>(dinfo.off), dinfo.count,
                             static_cast<uint32_t>(dinfo.subnet), row};
    f.write(reinterpret_cast<const char*>(hdr), sizeof(hdr));
    f.write(reinterpret_cast<const char*>(host_pool.data() + dinfo.off * kImg),
            static_cast<std::streamsize>(dinfo.count * kImg));
    f.write(reinterpret_cast<const char*>(dump_logits.data()),
            static_cast<std::streamsize>(dinfo.count * 1000 * sizeof(float)));
  }
  json j{{"mode", "serve"}, {"workers", workers}, {"gpus", ndev}, {"catalog", arg(a, "catalog", "")},
         {"load_fraction_of_sub0_capacity", load}, {"sub0_capacity_qps", cap0}, {"slo_us", slo},
         {"cv2", cv2}, {"duration_s", duration}, {"actuation", act}, {"actuation_charged_us", act_us},
         {"payload", "device-resident pool of 256 synthetic uint8 224x224 images (ssn_rng.h)"},
         {"runs", runs}, {"pass", ok}};
  std::cout << j.dump() << std::endl;
  return 0;
}

// ---------------------------------------------------------------- memory
// Weight-slice bytes of a subnet extracted as a standalone model (bf16
// weights + fp32 biases of its active slices, plus its BN scale/shift).
double extracted_bytes(const servesim::SubnetConfig& cfg) {
  ssn::CfgView v(cfg);
  ssn_supernet_desc d = r50_desc(64);
  std::vector<ssn_op_info> ops(512);
  uint32_t n = 0;
  ssn::check(ssn_plan_ops(&d, &v.c, ops.data(), 512, &n));
  double bytes = 0;
  for (uint32_t k = 0; k < n; ++k) {
    const auto& o = ops[k];
    if (!o.active) continue;
    if (o.kind == 1) bytes += 2.0 * o.cout * o.k * o.k * (o.depthwise ? 1 : o.cin) + 8.0 * o.cout;
    if (o.kind == 5) bytes += 2.0 * o.cout * o.cin + 4.0 * o.cout;
  }
  return bytes;
}

int cmd_memory(const std::map<std::string, std::string>& a) {
  const int many = std::stoi(arg(a, "many", "500"));
  ssn::Engine eng(std::stoi(arg(a, "device", "0")), r50_desc(64));
  std::vector<double> widths;
  double extracted6 = 0;
  for (int i = 0; i < 6; ++i) {
    const auto c = ofa_r50(kCatalog[i].d, kCatalog[i].e, kCatalog[i].w);
    eng.register_subnet(static_cast<uint32_t>(i), c);
    widths.push_back(c.mean_width_multiplier());
    extracted6 += extracted_bytes(c);
  }
  const ssn_stats s6 = eng.stats();
  servesim::MemorySpec spec;  // profile.hpp:512-516, filled with measured bytes
  spec.shared_weight_bytes = s6.weight_bytes;
  spec.per_subnet_stat_bytes = s6.norm_table_bytes / 6;
  spec.subnet_count = 6;
  const auto fp6 = servesim::memory_footprint(spec, widths);
  // `many` random OFA-R50 subnets registered at once ("simultaneous
  // actuation of 500 subnets"): per-block d / e / w drawn from the OFA lists
  std::mt19937_64 rng(1234);
  double stat_sum = 0, extracted_many = 0;
  for (int i = 0; i < many; ++i) {
    servesim::SubnetConfig c;  // (its members default to one-element lists)
    c.depth_flags.clear();
    c.expand_ratios.clear();
    c.width_multipliers.clear();
    c.depth_flags.push_back(rng() & 1);
    for (int b = 0; b < 8; ++b) c.depth_flags.push_back(rng() & 1);
    for (int b = 0; b < 18; ++b) c.expand_ratios.push_back(kExpands[rng() % 3]);
    for (int b = 0; b < 6; ++b) c.width_multipliers.push_back(kWidths[rng() % 3]);
    eng.register_subnet(static_cast<uint32_t>(6 + i), c);
    stat_sum += static_cast<double>(eng.stat_count(c)) * 2 * sizeof(float);
    extracted_many += extracted_bytes(c);
  }
  const ssn_stats sm = eng.stats();
  const double row_many = static_cast<double>(sm.norm_table_bytes - s6.norm_table_bytes) / many;
  servesim::MemorySpec spec_m = spec;
  spec_m.per_subnet_stat_bytes = static_cast<uint64_t>(row_many);
  spec_m.subnet_count = many;
  const auto fpm = servesim::memory_footprint(spec_m);
  json j{{"mode", "memory"},
         {"memory_spec_6", {{"shared_weight_bytes", spec.shared_weight_bytes},
                            {"per_subnet_stat_bytes", spec.per_subnet_stat_bytes},
                            {"subnet_count", spec.subnet_count}}},
         {"reference_memory_footprint_6", {{"supernet_bytes", fp6.supernet_bytes},
                                           {"individual_bytes_estimate", fp6.individual_bytes_estimate},
                                           {"stat_fraction", fp6.stat_fraction}}},
         {"measured_extracted_individual_bytes_6", extracted6},
         {"individual_over_supernet_6", extracted6 / static_cast<double>(fp6.supernet_bytes)},
         {"memory_spec_many", {{"shared_weight_bytes", spec_m.shared_weight_bytes},
                               {"per_subnet_stat_bytes", spec_m.per_subnet_stat_bytes},
                               {"subnet_count", spec_m.subnet_count}}},
         {"reference_memory_footprint_many", {{"supernet_bytes", fpm.supernet_bytes},
                                              {"individual_bytes_estimate", fpm.individual_bytes_estimate},
                                              {"stat_fraction", fpm.stat_fraction}}},
         {"measured_extracted_individual_bytes_many", extracted_many},
         {"individual_over_supernet_many", extracted_many / static_cast<double>(fpm.supernet_bytes)},
         {"shared_over_stat_row_mean_mu_var", static_cast<double>(spec.shared_weight_bytes) / (stat_sum / many)},
         {"shared_over_folded_norm_row_mean", static_cast<double>(spec.shared_weight_bytes) / row_many},
         {"engine_norm_table_bytes_total", sm.norm_table_bytes},
         {"registered_subnets", sm.registered_subnets},
         {"paper_claims", {{"lower_memory", "up to 2.6x (PAPER.md:451, 524)"},
                           {"stat_vs_shared", "500x smaller (PAPER.md:406, 485)"}}}};
  std::cout << j.dump() << std::endl;
  return 0;
}

// ---------------------------------------------------------------- actuation
int cmd_actuation(const std::map<std::string, std::string>& a) {
  const servesim::Catalog cat = with_configs(servesim::pareto_filter(
      servesim::load_catalog(arg(a, "catalog", "catalog_b200.csv"))));
  ssn::Engine eng(std::stoi(arg(a, "device", "0")), r50_desc(cat.max_batch));
  eng.register_catalog(cat);
  uint8_t* dx = nullptr;
  const std::vector<uint8_t> pool = make_pool();
  cuda_check(cudaMalloc(&dx, kImg), "cudaMalloc");
  cuda_check(cudaMemcpy(dx, pool.data(), kImg, cudaMemcpyHostToDevice), "upload");
  const json act = measure_actuation(eng, dx);
  cudaFree(dx);
  const Micros measured = static_cast<Micros>(std::ceil(act["switch_overhead_us"].get<double>() +
                                                        act["host_actuate_us_median"].get<double>()));
  const double cap0 = servesim::sustainable_qps(cat, cat.at(0).id, 1);
  const Micros slo = static_cast<Micros>(std::stod(arg(a, "slo-factor", "3")) * cat.at(cat.size() - 1).max_latency());
  json runs = json::array();
  for (uint32_t w : {1u, 8u}) {
    for (double load : {0.2, 0.4}) {
      servesim::TraceSpec spec;
      spec.kind = servesim::TraceKind::Bursty;
      spec.base_rate = 0.2 * load * w * cap0;
      spec.variant_rate = 0.8 * load * w * cap0;
      spec.cv2 = 4;
      spec.duration_s = std::stod(arg(a, "duration", "10"));
      spec.slo_us = slo;
      spec.seed = 7;
      const auto trace = servesim::generate_trace(spec);
      json row{{"workers", w}, {"load", load}, {"queries", trace.queries.size()}};
      for (Micros act_us : {Micros{0}, measured, Micros{100000}}) {
        servesim::SimConfig sc;
        sc.worker_count = w;
        sc.actuation_delay_us = act_us;
        sc.policy = servesim::PolicyKind::slackfit();
        const auto rep = servesim::run(trace, cat, sc);
        row["actuation_" + std::to_string(act_us) + "us"] = {
            {"slo_attainment", rep.aggregates.slo_attainment},
            {"mean_serving_accuracy", rep.aggregates.mean_serving_accuracy.value_or(0.0)}};
      }
      runs.push_back(row);
    }
  }
  json j{{"mode", "actuation"}, {"measured", act}, {"measured_charge_us", measured}, {"slo_us", slo},
         {"sub0_capacity_qps", cap0}, {"runs", runs},
         {"note", "servesim::run (simcore.hpp:129) on the B200 catalog; actuation 0 = ideal SubNetAct, "
                  "measured = this engine, 100000 = model switching (SPEC.md:343)"}};
  std::cout << j.dump() << std::endl;
  return 0;
}

// ---------------------------------------------------------------- simulate
// The reference router's decisions for a bursty trace on `workers` replicas
// (servesim::run, simcore.hpp:129, with its DispatchLog): one TSV row per
// dispatch "worker subnet_index actual_count profiled_batch start_us
// predicted_us", for bench.py's multi-replica SlackFit replay.  No engine.
int cmd_simulate(const std::map<std::string, std::string>& a) {
  const servesim::Catalog cat = servesim::pareto_filter(
      servesim::load_catalog(arg(a, "catalog", "catalog_b200.csv")));
  const uint32_t workers = std::stoul(arg(a, "workers", "1"));
  const double load = std::stod(arg(a, "load", "0.3"));
  const double cap0 = servesim::sustainable_qps(cat, cat.at(0).id, 1);
  servesim::TraceSpec spec;
  spec.kind = servesim::TraceKind::Bursty;
  spec.base_rate = 0.2 * load * workers * cap0;
  spec.variant_rate = 0.8 * load * workers * cap0;
  spec.cv2 = std::stod(arg(a, "cv2", "4"));
  spec.duration_s = std::stod(arg(a, "duration", "1"));
  spec.slo_us = static_cast<Micros>(std::stod(arg(a, "slo-factor", "3")) * cat.at(cat.size() - 1).max_latency());
  spec.seed = std::stoull(arg(a, "seed", "7"));
  const servesim::Trace trace = servesim::generate_trace(spec);
  servesim::SimConfig sc;
  sc.worker_count = workers;
  sc.actuation_delay_us = std::stoull(arg(a, "actuation-us", "1"));
  sc.policy = servesim::PolicyKind::slackfit();
  servesim::DispatchLog log;
  const servesim::SimReport rep = servesim::run(trace, cat, sc, &log);
  std::ofstream out(arg(a, "log", "dispatch.tsv"));
  for (const auto& r : log)
    out << r.worker << '\t' << r.subnet_index << '\t' << r.actual_count << '\t' << r.profiled_batch
        << '\t' << r.start_us << '\t' << r.predicted_latency_us << '\n';
  json j = servesim::report_to_json(rep);
  j["mode"] = "simulate";
  j["dispatches"] = log.size();
  j["lambda_qps"] = load * workers * cap0;
  j["sub0_capacity_qps"] = cap0;
  std::cout << j.dump() << std::endl;
  return 0;
}

}  // namespace

int main(int argc, char** argv) try {
  if (argc < 2) {
    std::cerr << "usage: serve_live profile|serve|memory|actuation [--key value ...]\n";
    return 2;
  }
  const std::string cmd = argv[1];
  const auto a = parse_args(argc, argv, 2);
  if (cmd == "profile") return cmd_profile(a);
  if (cmd == "serve") return cmd_serve(a);
  if (cmd == "memory") return cmd_memory(a);
  if (cmd == "actuation") return cmd_actuation(a);
  if (cmd == "simulate") return cmd_simulate(a);
  std::cerr << "unknown mode " << cmd << "\n";
  return 2;
} catch (const std::exception& e) {
  std::cerr << "error: " << e.what() << '\n';
  return 2;
}
