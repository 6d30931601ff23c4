// Drop-in for the control plane of agq/dbca.hpp + agq/layers.hpp: the DBCA
// per-stage bit-width planner (/root/reference/proj/include/agq/dbca.hpp:
// 13-177) and the activation-storage policy (layers.hpp:15-93), without the
// Eigen toy layer. plan_bit_widths runs in libagq_cuda.so (host code).
#pragma once

#include <algorithm>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../agq_cuda.h"
#include "quantize.hpp"

namespace agq {

struct PipelineConfig {
  int n_stages = 1;
  int micro_batches = 8;
  int interleave = 2;

  void check() const {
    std::vector<int> c(std::max(n_stages, 1));
    detail::throw_status(agq_stored_activation_counts(n_stages, micro_batches, interleave, c.data()));
  }
};

inline std::vector<int> stored_activation_counts(const PipelineConfig& cfg) {
  std::vector<int> c(std::max(cfg.n_stages, 1));
  detail::throw_status(
      agq_stored_activation_counts(cfg.n_stages, cfg.micro_batches, cfg.interleave, c.data()));
  c.resize(cfg.n_stages);
  return c;
}

struct StagePlan {
  int stage_index = 0;
  int stored_minibatches = 0;
  double raw_bits = 4.0;
  int assigned_bits = 4;
};

struct BitWidthPlan {
  int n_stages = 1;
  std::vector<StagePlan> stages;

  std::vector<int> assigned() const {
    std::vector<int> out;
    for (const auto& s : stages) out.push_back(s.assigned_bits);
    return out;
  }
};

inline BitWidthPlan plan_bit_widths(const PipelineConfig& cfg) {
  const int n = std::max(cfg.n_stages, 1);
  std::vector<int> counts(n), bits(n);
  std::vector<double> raw(n);
  detail::throw_status(agq_plan_bit_widths(cfg.n_stages, cfg.micro_batches, cfg.interleave,
                                           counts.data(), raw.data(), bits.data()));
  BitWidthPlan p;
  p.n_stages = cfg.n_stages;
  for (int i = 0; i < cfg.n_stages; ++i) p.stages.push_back({i + 1, counts[i], raw[i], bits[i]});
  return p;
}

struct StageMemory {
  int stage_index = 0;
  double bytes = 0.0;
  double budget_bytes = 0.0;
};

struct PeakMemoryCheck {
  std::vector<StageMemory> stages;
  double budget_bytes = 0.0;
  double slack_bytes = 0.0;
  bool pass = false;
  std::string note;
};

// Stage i stores N_i * bits_i / 16 of a 16-bit mini-batch; the budget is the
// most loaded stage at 4 bits plus one bit per element of rounding slack.
inline PeakMemoryCheck peak_memory_check(const BitWidthPlan& plan, double bytes_per_minibatch_at_16bit) {
  if (plan.stages.empty()) throw std::invalid_argument("empty plan");
  const double per_bit = bytes_per_minibatch_at_16bit / 16.0;
  int most = 0;
  for (const auto& s : plan.stages) most = std::max(most, s.stored_minibatches);
  PeakMemoryCheck out;
  out.budget_bytes = most * 4.0 * per_bit;
  out.pass = true;
  for (const auto& s : plan.stages) {
    const double slack = s.stored_minibatches * per_bit;
    const StageMemory m{s.stage_index, s.stored_minibatches * s.assigned_bits * per_bit,
                        out.budget_bytes + slack};
    out.slack_bytes = std::max(out.slack_bytes, slack);
    out.pass = out.pass && !(m.bytes > m.budget_bytes);
    out.stages.push_back(m);
  }
  out.note = "budget is the most loaded stage at 4 bits, plus a rounding allowance of one bit "
             "per element on the stage under test";
  return out;
}

struct PlanReuseCheck {
  std::vector<int> applied_bits;
  double peak = 0.0;
  double uniform4_peak = 0.0;
  bool pass = false;
};

inline PlanReuseCheck plan_reuse_check(const PipelineConfig& low, const PipelineConfig& high) {
  if (low.n_stages > high.n_stages)
    throw std::invalid_argument("plan reuse goes from fewer stages to more stages");
  const auto lp = plan_bit_widths(low);
  const auto hc = stored_activation_counts(high);
  PlanReuseCheck out;
  out.applied_bits.assign(hc.size(), 4);
  for (int i = 0; i < low.n_stages; ++i)  // anchored at the lightly loaded end
    out.applied_bits[hc.size() - 1 - i] = lp.stages[low.n_stages - 1 - i].assigned_bits;
  for (std::size_t i = 0; i < hc.size(); ++i) {
    out.peak = std::max(out.peak, static_cast<double>(hc[i]) * out.applied_bits[i]);
    out.uniform4_peak = std::max(out.uniform4_peak, hc[i] * 4.0);
  }
  out.pass = true;
  for (std::size_t i = 0; i < hc.size(); ++i)
    if (static_cast<double>(hc[i]) * out.applied_bits[i] > out.uniform4_peak + hc[i]) out.pass = false;
  return out;
}

enum class LayerRole { RmsNorm, QkvProj, Attention, OutProj, Ffn1, SiluMul, Ffn2 };

inline const char* layer_role_name(LayerRole r) {
  static const char* kNames[] = {"rmsnorm", "qkv_proj", "attention", "out_proj",
                                 "ffn1", "silu_mul", "ffn2"};
  return kNames[static_cast<int>(r)];
}

enum class SaveStrategy { RecomputeIntermediates, CacheIntermediates, NoQuant };

struct PolicyEntry {
  int bit_width = 0;  // 0 = full precision
  SaveStrategy strategy = SaveStrategy::NoQuant;
};

struct ActivationPolicy {
  std::map<LayerRole, PolicyEntry> entries;

  static ActivationPolicy all_full() {
    ActivationPolicy p;
    for (int r = 0; r <= static_cast<int>(LayerRole::Ffn2); ++r)
      p.entries[static_cast<LayerRole>(r)] = {0, SaveStrategy::NoQuant};
    return p;
  }

  // bits on every role with recomputation, except full-precision attention
  // internals and a quantized cached out-projection input.
  static ActivationPolicy agoq_default(int bits = 4) {
    ActivationPolicy p;
    for (int r = 0; r <= static_cast<int>(LayerRole::Ffn2); ++r)
      p.entries[static_cast<LayerRole>(r)] = {bits, SaveStrategy::RecomputeIntermediates};
    p.entries[LayerRole::Attention] = {0, SaveStrategy::NoQuant};
    p.entries[LayerRole::OutProj] = {bits, SaveStrategy::CacheIntermediates};
    p.validate();
    return p;
  }

  const PolicyEntry& at(LayerRole role) const {
    const auto it = entries.find(role);
    if (it == entries.end())
      throw std::runtime_error(std::string("policy has no entry for role ") + layer_role_name(role));
    return it->second;
  }

  void validate() const {
    for (const auto& kv : entries) {
      const PolicyEntry& e = kv.second;
      if (e.bit_width != 0 && (e.bit_width < 4 || e.bit_width > 8))
        throw std::invalid_argument("policy bit width must be FULL or in [4,8]");
      if (e.strategy == SaveStrategy::NoQuant && e.bit_width != 0)
        throw std::invalid_argument("NO_QUANT entries store full precision");
    }
  }
};

inline ActivationPolicy stage_policy(const BitWidthPlan& plan, int stage_index) {
  for (const auto& s : plan.stages)
    if (s.stage_index == stage_index) return ActivationPolicy::agoq_default(s.assigned_bits);
  throw std::invalid_argument("no such stage in plan");
}

}  // namespace agq
