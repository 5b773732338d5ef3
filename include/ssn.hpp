// ssn.hpp — C++ host wrapper over the SubNetAct C-ABI (include/ssn.h).
//
// Mirrors the reference's conventions so a servesim worker can call it as-is:
//  * errors are rethrown as the exception types the reference uses
//    (std::invalid_argument, std::out_of_range, std::runtime_error, std::logic_error;
//    reference profile.hpp:40-53, 79-80, policy.hpp:92-98);
//  * `register_subnet` / `register_catalog` accept servesim::SubnetConfig /
//    servesim::Catalog (or anything with the same members) without this header
//    depending on the reference headers;
//  * one Engine per GPU, driven by one worker thread (serve_runtime.hpp:1-6).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "ssn.h"

namespace ssn {

inline void check(int rc) {
  if (rc == SSN_OK) return;
  const std::string msg = ssn_last_error();
  switch (rc) {
    case SSN_E_INVALID: throw std::invalid_argument(msg);
    case SSN_E_RANGE: throw std::out_of_range(msg);
    case SSN_E_STATE: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// servesim::SubnetConfig has no kernel list (profile.hpp:28-54); a config type
// that carries one (`kernel_sizes`, OFA-MBv3) passes it through.
template <class T, class = void>
struct has_kernel_sizes : std::false_type {};
template <class T>
struct has_kernel_sizes<T, std::void_t<decltype(std::declval<const T&>().kernel_sizes)>>
    : std::true_type {};

// Owning view of a control tuple in C-ABI form.
struct CfgView {
  std::vector<uint8_t> d;
  std::vector<double> e, w;
  std::vector<uint32_t> k;
  ssn_subnet_cfg c{};
  template <class Cfg>
  explicit CfgView(const Cfg& cfg) {
    for (bool f : cfg.depth_flags) d.push_back(f ? 1 : 0);
    e.assign(cfg.expand_ratios.begin(), cfg.expand_ratios.end());
    w.assign(cfg.width_multipliers.begin(), cfg.width_multipliers.end());
    if constexpr (has_kernel_sizes<Cfg>::value)  // elastic-kernel supernets (OFA-MBv3)
      for (auto ks : cfg.kernel_sizes) k.push_back(static_cast<uint32_t>(ks));
    c.depth_flags = d.data();
    c.n_depth = static_cast<uint32_t>(d.size());
    c.expand_ratios = e.data();
    c.n_expand = static_cast<uint32_t>(e.size());
    c.width_multipliers = w.data();
    c.n_width = static_cast<uint32_t>(w.size());
    c.kernel_sizes = k.empty() ? nullptr : k.data();
    c.n_kernel = static_cast<uint32_t>(k.size());
  }
};

class Engine {
 public:
  Engine(int device, const ssn_supernet_desc& desc, const void* host_weights = nullptr,
         uint64_t host_weight_bytes = 0) {
    check(ssn_create(device, &desc, host_weights, host_weight_bytes, &h_));
  }
  ~Engine() { ssn_destroy(h_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  template <class Cfg>
  uint64_t stat_count(const Cfg& cfg) const {
    CfgView v(cfg);
    uint64_t n = 0;
    check(ssn_subnet_stat_count(h_, &v.c, &n));
    return n;
  }

  // subnet_index = position in the pareto-sorted catalog (policy.hpp:187-190)
  template <class Cfg>
  void register_subnet(uint32_t subnet_index, const Cfg& cfg, const float* bn_mean = nullptr,
                       const float* bn_var = nullptr) {
    CfgView v(cfg);
    check(ssn_register_subnet(h_, subnet_index, &v.c, bn_mean, bn_var));
  }

  // Registers every record of a (pareto) servesim::Catalog by index and builds
  // the graph segments for its batch grid (Catalog::batch_sizes, profile.hpp:164).
  template <class Catalog>
  void register_catalog(const Catalog& catalog) {
    for (std::size_t i = 0; i < catalog.subnets.size(); ++i)
      register_subnet(static_cast<uint32_t>(i), catalog.subnets[i].config);
    std::vector<uint32_t> grid;
    for (auto b : catalog.batch_sizes()) grid.push_back(static_cast<uint32_t>(b));
    prepare(grid);
  }

  void prepare(const std::vector<uint32_t>& batch_grid) {
    check(ssn_prepare(h_, batch_grid.data(), static_cast<uint32_t>(batch_grid.size())));
  }
  void actuate(uint32_t subnet_index) { check(ssn_actuate(h_, subnet_index)); }
  void forward(const void* images, uint32_t count, uint32_t profiled_batch, float* logits,
               void* stream = nullptr) {
    check(ssn_forward(h_, images, count, profiled_batch, logits, stream));
  }
  void synchronize(void* stream = nullptr) { check(ssn_synchronize(h_, stream)); }
  double profile_latency_us(uint32_t subnet_index, uint32_t batch, uint32_t iters = 20) {
    double us = 0;
    check(ssn_profile_latency(h_, subnet_index, batch, iters, &us));
    return us;
  }
  ssn_stats stats() const {
    ssn_stats s{};
    check(ssn_query(h_, &s));
    return s;
  }
  ssn_engine* handle() const { return h_; }

 private:
  ssn_engine* h_ = nullptr;
};

// The worker body of serve_runtime.hpp:161-172 with the sleep replaced:
// actuate the dispatched subnet in place, run the (clamped) batch, wait.
// `images` holds cmd.batch's payload (the reference's Query has none,
// edf_queue.hpp:16-20; see DESIGN.md §3.3 for the synthetic payload).
struct EngineWorker {
  Engine& engine;
  template <class DispatchCmd>
  void run(const DispatchCmd& cmd, uint32_t profiled_batch, const void* images, float* logits) {
    engine.actuate(static_cast<uint32_t>(cmd.subnet_index));
    engine.forward(images, static_cast<uint32_t>(cmd.batch.queries.size()), profiled_batch, logits);
    engine.synchronize();
  }
};

}  // namespace ssn
