// ssn_serve.hpp — servesim's live mode with SubNetAct engines as its workers.
//
// The reference's live runtime (`servesim::serve`, serve_runtime.hpp:113-438)
// hard-codes its worker body as a sleep for the profiled latency
// (serve_runtime.hpp:161-172, sleep at :167).  This header is the same live
// runtime with that body replaced by real inference: each worker thread owns
// one ssn::Engine (one GPU), actuates the dispatched subnet in place and runs
// the clamped batch, then reports the REAL completion time.
//
// Everything the dispatcher decides with is the reference's own code, used
// unmodified: EdfQueue (edf_queue.hpp), decide / clamp_decision /
// build_buckets / min_feasible_latency (policy.hpp, profile.hpp), the message
// types serve_detail::Channel / FreeMsg / DispatchCmd (serve_runtime.hpp:48-
// 104), DispatchLog (simcore.hpp:56-70) and the report (metrics.hpp:91-106).
// The dispatch loop below restates serve_runtime.hpp:216-388 with identical
// decisions (single dispatcher thread, lowest-id idle worker, the same
// drop / decide / clamp order, the same actuation bookkeeping, the same
// fault handling); what differs is only what a worker does with a command.
//
// Not restated: the 100 ms dynamics reconstruction (serve_runtime.hpp:394-
// 433) — report.dynamics stays empty; aggregates / outcomes / the dispatch
// log / pacing_overrun / diverged are produced exactly as the reference does.
//
// Threading: the dispatcher never touches an engine; engine i is driven only
// by worker thread i (include/ssn.h, "one engine per GPU, one worker thread").
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <thread>
#include <variant>
#include <vector>

#include "servesim/serve_runtime.hpp"
#include "ssn.hpp"

namespace ssn {

// Per-dispatch record a worker keeps (what the engine actually did).
struct LiveDispatch {
  uint32_t worker = 0;
  std::size_t subnet_index = 0;
  uint32_t count = 0;           // ClampedDispatch::actual_count
  uint32_t profiled_batch = 0;  // graph key (ceil_entry, profile.hpp:92-98)
  servesim::Micros start_us = 0;       // worker picked the command up
  servesim::Micros completion_us = 0;  // engine finished (FreeMsg time)
  servesim::Micros predicted_us = 0;   // catalog latency of the clamped batch
  double actuate_us = 0;               // host cost of ssn_actuate
  bool switched = false;               // subnet differs from the previous one
};

// Supplies a batch's images (`Batch` carries no payload, edf_queue.hpp:16-31)
// and, optionally, where its logits go (nullptr: keep them on the device).
struct Payload {
  std::function<const void*(const servesim::Batch&, uint32_t worker, std::size_t subnet)> images;
  std::function<float*(const servesim::Batch&, uint32_t worker, std::size_t subnet)> logits;
};

struct LiveResult {
  servesim::SimReport report;
  std::vector<LiveDispatch> dispatches;  // in completion order per worker
  double wall_s = 0;
};

// servesim::serve (serve_runtime.hpp:113) with engine-backed workers.
// `engines[i]` serves worker i; config.worker_count must equal engines.size().
// config.actuation_delay_us is NOT slept: actuation is the engine's real
// cost; the value is only echoed and used for the dispatch log's
// actuation_us bookkeeping exactly as the reference computes it.
inline LiveResult serve_engines(const servesim::Trace& trace, const servesim::Catalog& catalog,
                                const servesim::ServeConfig& config,
                                const std::vector<Engine*>& engines, const Payload& payload,
                                servesim::DispatchLog* log = nullptr) {
  using namespace servesim;
  using namespace servesim::serve_detail;
  using Clock = std::chrono::steady_clock;
  if (engines.size() != config.worker_count)
    throw std::invalid_argument("serve_engines: one engine per worker");

  SimConfig sim_like;  // the reference validates live configs this way (:124-131)
  sim_like.worker_count = config.worker_count;
  sim_like.actuation_delay_us = config.actuation_delay_us;
  sim_like.dispatch_overhead_us = config.dispatch_overhead_us;
  sim_like.policy = config.policy;
  sim_like.bucket_count = config.bucket_count;
  sim_like.fault_schedule = config.fault_schedule;
  sim_like.validate(catalog);
  const BucketTable buckets = build_buckets(catalog, config.bucket_count);
  const Micros floor_us = min_feasible_latency(config.policy, catalog) + config.dispatch_overhead_us;

  LiveResult res;
  SimReport& report = res.report;
  report.config_echo = {{"mode", "serve_engines"},
                        {"policy", to_string(config.policy)},
                        {"workers", config.worker_count},
                        {"actuation_delay_us", config.actuation_delay_us},
                        {"dispatch_overhead_us", config.dispatch_overhead_us},
                        {"bucket_count", config.bucket_count},
                        {"trace_spec", trace_spec_to_json(trace.spec)},
                        {"trace_queries", trace.queries.size()}};

  // every thread parks on its channel before the first arrival (:145)
  const auto t0 = Clock::now() + std::chrono::milliseconds(100);
  auto now_us = [&]() -> Micros {
    const auto d = std::chrono::duration_cast<std::chrono::microseconds>(Clock::now() - t0).count();
    return d < 0 ? 0 : static_cast<Micros>(d);
  };

  Channel<RouterMsg> inbox;
  std::vector<std::unique_ptr<Channel<DispatchCmd>>> chans;
  for (uint32_t i = 0; i < config.worker_count; ++i) chans.push_back(std::make_unique<Channel<DispatchCmd>>());
  std::vector<std::vector<LiveDispatch>> per_worker(config.worker_count);

  // ---- workers: the reference's sleep (:167) becomes actuate + forward
  std::vector<std::thread> threads;
  for (uint32_t i = 0; i < config.worker_count; ++i) {
    threads.emplace_back([&, i] {
      Engine& eng = *engines[i];
      std::optional<std::size_t> current;
      for (;;) {
        auto cmd = chans[i]->pop();
        if (!cmd || cmd->stop) return;
        LiveDispatch rec;
        rec.worker = i;
        rec.subnet_index = cmd->subnet_index;
        rec.count = cmd->batch.size();
        const auto entry = catalog.at(cmd->subnet_index).ceil_entry(rec.count);
        rec.profiled_batch = entry.batch;
        rec.predicted_us = entry.latency_us;
        rec.switched = !current || *current != cmd->subnet_index;
        current = cmd->subnet_index;
        rec.start_us = now_us();
        eng.actuate(static_cast<uint32_t>(cmd->subnet_index));
        rec.actuate_us = eng.stats().last_actuate_us;
        eng.forward(payload.images(cmd->batch, i, cmd->subnet_index), rec.count, rec.profiled_batch,
                    payload.logits ? payload.logits(cmd->batch, i, cmd->subnet_index) : nullptr);
        eng.synchronize();
        rec.completion_us = now_us();
        per_worker[i].push_back(rec);
        inbox.push(FreeMsg{i, rec.completion_us, std::move(cmd->batch), cmd->subnet_index});
      }
    });
  }

  // ---- client: real-time replay of the trace (:174-183)
  std::thread client([&] {
    Micros late = 0;
    for (const auto& q : trace.queries) {
      std::this_thread::sleep_until(t0 + std::chrono::microseconds(q.arrival_us));
      const Micros t = now_us();
      if (t > q.arrival_us) late = std::max(late, t - q.arrival_us);
      inbox.push(EnqueueMsg{q, t});
    }
    inbox.push(ClientDoneMsg{late});
  });

  // ---- dispatcher: sole owner of the queue and worker bookkeeping
  struct Slot {
    bool busy = false, alive = true, doomed = false;
    std::optional<std::size_t> current_subnet;
  };
  std::vector<Slot> slots(config.worker_count);
  std::vector<FaultSpec> faults = config.fault_schedule;
  std::sort(faults.begin(), faults.end(),
            [](const FaultSpec& a, const FaultSpec& b) { return a.time_us < b.time_us; });
  std::size_t next_fault = 0, in_flight = 0, dropped = 0, backlog = 0;
  bool client_done = false;
  Micros max_late = 0;
  EdfQueue queue;

  auto drop = [&](const Query& q) {
    report.outcomes.push_back({q.id, OutcomeKind::Dropped, 0.0, 0, q.deadline_us});
    ++dropped;
  };
  auto first_idle = [&]() -> std::optional<uint32_t> {  // lowest-id idle worker (:216-221)
    for (uint32_t w = 0; w < slots.size(); ++w)
      if (slots[w].alive && !slots[w].busy) return w;
    return std::nullopt;
  };
  auto schedule = [&] {  // try_schedule (:250-305)
    const Micros now = now_us();
    while (!queue.empty()) {
      const auto w = first_idle();
      if (!w) return;
      for (const auto& q : queue.drop_expired(now, floor_us)) drop(q);
      if (queue.empty()) return;
      const SlackMicros slack =
          *queue.peek_slack(now) - static_cast<SlackMicros>(config.dispatch_overhead_us);
      const auto d = decide(config.policy, slack, queue.size(), buckets, catalog);
      if (!d) {
        drop(queue.take_batch(1).queries.front());
        continue;
      }
      const auto c = clamp_decision(*d, queue.size(), catalog);
      Batch batch = queue.take_batch(c.actual_count);
      Slot& s = slots[*w];
      const Micros act =
          (s.current_subnet && *s.current_subnet == d->subnet_index) ? 0 : config.actuation_delay_us;
      s.busy = true;
      s.current_subnet = d->subnet_index;
      ++in_flight;
      if (log) {
        DispatchRecord r;
        r.start_us = now;
        r.worker = *w;
        r.subnet_index = d->subnet_index;
        r.accuracy = catalog.at(d->subnet_index).accuracy;
        r.actual_count = c.actual_count;
        r.profiled_batch = c.profiled_batch;
        r.predicted_latency_us = c.latency_us;
        r.actuation_us = act;
        r.batch_arrival_us = batch.arrival_us;
        r.batch_deadline_us = batch.deadline_us;
        for (const auto& q : batch.queries) r.query_ids.push_back(q.id);
        log->push_back(std::move(r));
      }
      chans[*w]->push(DispatchCmd{std::move(batch), d->subnet_index, act + c.latency_us, false});
    }
  };

  const auto wall0 = Clock::now();
  for (;;) {
    const auto until = next_fault < faults.size()
                           ? t0 + std::chrono::microseconds(faults[next_fault].time_us)
                           : Clock::now() + std::chrono::milliseconds(50);
    auto msg = inbox.pop_until(until);
    const Micros now = now_us();
    for (; next_fault < faults.size() && faults[next_fault].time_us <= now; ++next_fault) {
      Slot& s = slots[faults[next_fault].worker];
      if (!s.alive) continue;
      if (s.busy)
        s.doomed = true;  // dies when its batch completes (:236-249)
      else
        s.alive = false;
    }
    if (msg) {
      if (auto* e = std::get_if<EnqueueMsg>(&*msg)) {
        queue.enqueue(e->query);
        report.max_queue_depth = std::max(report.max_queue_depth, queue.size());
        backlog = std::max(backlog, queue.size() + dropped);
      } else if (auto* f = std::get_if<FreeMsg>(&*msg)) {
        const double acc = catalog.at(f->subnet_index).accuracy;
        for (const auto& q : f->batch.queries) {
          const bool hit = f->completion_us <= q.deadline_us;  // simcore.hpp:348
          report.outcomes.push_back({q.id, hit ? OutcomeKind::Hit : OutcomeKind::Miss,
                                     hit ? acc : 0.0, f->completion_us, q.deadline_us});
        }
        if (log)
          for (auto& r : *log)
            if (r.worker == f->worker && r.completion_us == 0) {
              r.completion_us = f->completion_us;
              break;
            }
        Slot& s = slots[f->worker];
        s.busy = false;
        if (s.doomed) s.alive = s.doomed = false;
        --in_flight;
      } else if (auto* done = std::get_if<ClientDoneMsg>(&*msg)) {
        client_done = true;
        max_late = done->max_lateness_us;
      }
    }
    schedule();
    if (client_done && in_flight == 0) {
      if (queue.empty()) break;
      bool any_alive = false;
      for (const auto& s : slots) any_alive |= s.alive;
      if (!any_alive) {
        while (!queue.empty()) drop(queue.take_batch(1).queries.front());
        break;
      }
    }
  }
  for (auto& ch : chans) ch->push(DispatchCmd{{}, 0, 0, true});
  for (auto& t : threads) t.join();
  client.join();
  res.wall_s = std::chrono::duration<double>(Clock::now() - wall0).count();

  report.pacing_overrun = max_late > config.pacing_tolerance_us;
  if (trace.queries.size() >= 2) {  // the reference's divergence rule (:371-392)
    const double span = static_cast<double>(trace.last_arrival_us() - trace.queries.front().arrival_us) / 1e6;
    if (span > 0.0) {
      double slo = 0.0;
      for (const auto& q : trace.queries) slo += static_cast<double>(q.deadline_us - q.arrival_us);
      const double lambda = static_cast<double>(trace.queries.size()) / span;
      report.diverged = static_cast<double>(backlog) >
                        50.0 * lambda * slo / static_cast<double>(trace.queries.size()) / 1e6;
    }
  }
  finalize_report(report);
  for (auto& v : per_worker) res.dispatches.insert(res.dispatches.end(), v.begin(), v.end());
  return res;
}

}  // namespace ssn
