// core.cpp -- host-side bookkeeping the serving loop needs: precision tags,
// cost model, the elastic KV block pool, the morphing controller, the
// LayerSwapper residency state, traces and metrics.  Each piece keeps the
// observable behaviour of its reference counterpart (file:line cited per
// function) because block tables, swap decisions and metric definitions must
// be bit-identical to the reference.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <numeric>
#include <random>
#include <sstream>
#include <stdexcept>
#include <unordered_set>

#include "host.hpp"

namespace morphserve {

// ---------------------------------------------------------------- precision
int precision_bits(Precision p) {
  static const int bits[4] = {16, 8, 4, 3};
  return bits[static_cast<int>(p)];
}
Precision precision_from_bits(int bits) {  // reference toy_model.cpp:20-28
  if (bits == 16) return Precision::kFull;
  if (bits == 8) return Precision::kQ8;
  if (bits == 4) return Precision::kQ4;
  if (bits == 3) return Precision::kQ3;
  throw std::invalid_argument("unsupported bit width: " + std::to_string(bits));
}
std::string precision_name(Precision p) {
  static const char* names[4] = {"full", "q8", "q4", "q3"};
  return names[static_cast<int>(p)];
}

// -------------------------------------------------------------- cost model
int64_t gib_to_bytes(double gib) { return static_cast<int64_t>(std::llround(gib * static_cast<double>(kGiB))); }

void SimModelConfig::validate() const {  // reference sim_config.cpp:13-22
  if (num_layers < 1) throw std::invalid_argument("model: num_layers must be >= 1");
  for (int64_t b : layer_bytes)
    if (b < 1) throw std::invalid_argument("model: layer byte sizes must be positive");
  for (int i = 0; i + 1 < 4; ++i)
    if (layer_bytes[i] < layer_bytes[i + 1])
      throw std::invalid_argument("model: layer bytes must be non-increasing with precision");
}

// reference sim_config.cpp:23-27: attention term first, then per-layer terms in order
double CostModel::decode_step_ms(const std::vector<Precision>& tags, int64_t batch_blocks) const {
  double ms = attn_ms_per_kv_block * static_cast<double>(batch_blocks);
  for (Precision t : tags) ms += decode_ms_per_layer[static_cast<int>(t)];
  return ms;
}
// reference sim_config.cpp:29-33
double CostModel::swap_duration_ms(int64_t variant_bytes) const {
  return swap_fixed_overhead_ms +
         static_cast<double>(variant_bytes) / (pcie_gib_per_s * static_cast<double>(kGiB)) * 1000.0;
}
void CostModel::validate() const {
  if (!(prefill_ms_per_token > 0.0)) throw std::invalid_argument("cost: prefill rate must be > 0");
  for (double v : decode_ms_per_layer)
    if (!(v > 0.0)) throw std::invalid_argument("cost: decode layer costs must be > 0");
  for (int i = 0; i + 1 < 4; ++i)
    if (decode_ms_per_layer[i] < decode_ms_per_layer[i + 1])
      throw std::invalid_argument("cost: decode cost must be non-increasing as precision drops");
  if (!(attn_ms_per_kv_block > 0.0)) throw std::invalid_argument("cost: attn term must be > 0");
  if (!(pcie_gib_per_s > 0.0)) throw std::invalid_argument("cost: pcie rate must be > 0");
  if (!(swap_fixed_overhead_ms > 0.0)) throw std::invalid_argument("cost: swap overhead must be > 0");
  if (max_batch_tokens < 1) throw std::invalid_argument("cost: max_batch_tokens must be >= 1");
}

// ----------------------------------------------------------- KV block pool
KvBlockPool::KvBlockPool(const KvConfig& config) : cfg_(config) {
  if (config.block_tokens < 1) throw std::invalid_argument("kv pool: block_tokens must be >= 1");
  if (config.block_bytes < 1) throw std::invalid_argument("kv pool: block_bytes must be >= 1");
  if (config.static_capacity_blocks < 1) throw std::invalid_argument("kv pool: static_capacity_blocks must be >= 1");
  capacity_ = config.static_capacity_blocks;
  free_.reserve(static_cast<size_t>(capacity_));
  while (next_id_ < capacity_) free_.push_back(next_id_++);  // ids 0..cap-1, top = cap-1
}

void KvBlockPool::admit(RequestId req) {
  auto ins = reqs_.try_emplace(req);
  if (!ins.second) throw std::invalid_argument("kv pool: request already admitted");
  ins.first->second.stamp = next_stamp_++;
}

int64_t KvBlockPool::blocks_needed_for(int64_t existing, int64_t grow) const {
  const int64_t bt = cfg_.block_tokens;
  return (existing + grow + bt - 1) / bt - (existing + bt - 1) / bt;
}

// all-or-nothing, pops from the top of the free stack (reference kv_pool.cpp:33-52)
std::optional<std::vector<BlockId>> KvBlockPool::alloc_for_tokens(RequestId req, int64_t new_tokens) {
  auto it = reqs_.find(req);
  if (it == reqs_.end()) throw std::invalid_argument("kv pool: unknown request in alloc");
  if (new_tokens < 1) throw std::invalid_argument("kv pool: new_tokens must be >= 1");
  const int64_t need = blocks_needed_for(it->second.tokens, new_tokens);
  if (need > free_blocks()) return std::nullopt;
  std::vector<BlockId> got(static_cast<size_t>(need));
  for (auto& id : got) {
    id = free_.back();
    free_.pop_back();
  }
  it->second.blocks.insert(it->second.blocks.end(), got.begin(), got.end());
  it->second.tokens += new_tokens;
  return got;
}

void KvBlockPool::drain_pending_detach() {  // reference kv_pool.cpp:54-64
  while (pending_detach_ > 0 && !free_.empty()) {
    retired_.push_back(free_.back());
    free_.pop_back();
    --pending_detach_;
    --capacity_;
    --attached_;
  }
}

int64_t KvBlockPool::release(RequestId req) {  // reference kv_pool.cpp:66-75
  auto it = reqs_.find(req);
  if (it == reqs_.end()) throw std::invalid_argument("kv pool: unknown request in release");
  const auto& blocks = it->second.blocks;
  const int64_t n = static_cast<int64_t>(blocks.size());
  free_.insert(free_.end(), blocks.begin(), blocks.end());
  reqs_.erase(it);
  drain_pending_detach();
  return n;
}

int64_t KvBlockPool::attach_blocks(int64_t n) {  // reference kv_pool.cpp:77-83
  if (n < 1) throw std::invalid_argument("kv pool: attach count must be >= 1");
  for (int64_t i = 0; i < n; ++i) free_.push_back(next_id_++);
  capacity_ += n;
  attached_ += n;
  return capacity_;
}

DetachResult KvBlockPool::detach_blocks(int64_t n) {  // reference kv_pool.cpp:85-100
  if (n < 1) throw std::invalid_argument("kv pool: detach count must be >= 1");
  if (n > attached_ - pending_detach_) throw std::invalid_argument("kv pool: detach exceeds attached extra blocks");
  const int64_t now = std::min<int64_t>(n, free_blocks());
  for (int64_t i = 0; i < now; ++i) {
    retired_.push_back(free_.back());
    free_.pop_back();
  }
  capacity_ -= now;
  attached_ -= now;
  pending_detach_ += n - now;
  return DetachResult{now, n - now, capacity_};
}

std::optional<RequestId> KvBlockPool::preempt_victim(const std::function<bool(RequestId)>& eligible) {
  // newest admission among the eligible (reference kv_pool.cpp:102-118)
  const Entry* best = nullptr;
  RequestId victim = -1;
  for (const auto& kv : reqs_) {
    if (!eligible(kv.first)) continue;
    if (!best || kv.second.stamp > best->stamp) {
      best = &kv.second;
      victim = kv.first;
    }
  }
  if (!best) return std::nullopt;
  release(victim);
  return victim;
}

int64_t KvBlockPool::tokens_of(RequestId req) const {
  auto it = reqs_.find(req);
  if (it == reqs_.end()) throw std::invalid_argument("kv pool: unknown request in tokens_of");
  return it->second.tokens;
}
int64_t KvBlockPool::blocks_of(RequestId req) const {
  auto it = reqs_.find(req);
  if (it == reqs_.end()) throw std::invalid_argument("kv pool: unknown request in blocks_of");
  return static_cast<int64_t>(it->second.blocks.size());
}
const std::vector<BlockId>& KvBlockPool::block_list(RequestId req) const {
  auto it = reqs_.find(req);
  if (it == reqs_.end()) throw std::invalid_argument("kv pool: unknown request in block_list");
  return it->second.blocks;
}
double KvBlockPool::usage_fraction() const {
  return capacity_ == 0 ? 0.0 : static_cast<double>(used_blocks()) / static_cast<double>(capacity_);
}
std::vector<BlockId> KvBlockPool::take_retired() {
  std::vector<BlockId> out;
  out.swap(retired_);
  return out;
}
void KvBlockPool::check_invariants() const {  // reference kv_pool.cpp:137-158
  std::unordered_set<BlockId> seen;
  int64_t held = 0;
  auto add = [&](BlockId id) {
    if (!seen.insert(id).second) throw std::logic_error("kv pool: duplicate block id");
  };
  for (BlockId id : free_) add(id);
  for (const auto& kv : reqs_) {
    held += static_cast<int64_t>(kv.second.blocks.size());
    for (BlockId id : kv.second.blocks) add(id);
  }
  if (free_blocks() + held != capacity_) throw std::logic_error("kv pool: free + allocated != capacity");
  if (capacity_ != cfg_.static_capacity_blocks + attached_)
    throw std::logic_error("kv pool: capacity != static + attached_extra");
  if (pending_detach_ < 0 || attached_ < 0) throw std::logic_error("kv pool: negative bookkeeping counter");
}

// -------------------------------------------------------------- controller
void ControllerConfig::validate(int num_layers) const {  // reference controller.cpp:8-24
  if (!enabled) return;
  if (!(kv_low > 0.0) || !(kv_low < kv_trigger) || !(kv_trigger <= 1.0))
    throw std::invalid_argument("controller: need 0 < kv_low < kv_trigger <= 1");
  if (!(queue_trigger_ms > 0.0)) throw std::invalid_argument("controller: queue trigger must be > 0");
  if (!(hold_ms > 0.0)) throw std::invalid_argument("controller: hold_ms must be > 0");
  if (swap_step < 1 || swap_step > max_swapped_layers || max_swapped_layers > num_layers)
    throw std::invalid_argument("controller: need 1 <= swap_step <= max_swapped_layers <= L");
  if (!(telemetry_window_ms > 0.0)) throw std::invalid_argument("controller: telemetry window must be > 0");
  if (target_bits != 8 && target_bits != 4 && target_bits != 3)
    throw std::invalid_argument("controller: target_bits must be one of 8, 4, 3");
}

ControllerConfig ControllerConfig::defaults_for(ControllerMode mode, int num_layers) {  // controller.cpp:26-40
  ControllerConfig c;
  c.enabled = true;
  c.mode = mode;
  const bool acc = mode == ControllerMode::kAccuracy;
  c.kv_trigger = acc ? 0.92 : 0.80;
  c.max_swapped_layers = std::max(1, acc ? num_layers / 4 : num_layers / 2);
  c.swap_step = acc ? 1 : std::min(2, std::max(1, num_layers / 2));
  return c;
}

void TelemetryWindow::push(const TelemetrySample& s) {  // controller.cpp:42-48
  last_ = s;
  samples_.push_back(s);
  while (!samples_.empty() && samples_.front().t_ms < s.t_ms - window_ms_) samples_.pop_front();
}
template <class Get>
double TelemetryWindow::mean(Get get) const {
  if (samples_.empty()) return get(last_);
  double sum = 0.0;
  for (const auto& s : samples_) sum += get(s);
  return sum / static_cast<double>(samples_.size());
}
double TelemetryWindow::mean_kv_usage() const { return mean([](const TelemetrySample& s) { return s.kv_usage; }); }
double TelemetryWindow::mean_queue_depth() const {
  return mean([](const TelemetrySample& s) { return s.queue_depth; });
}
double TelemetryWindow::mean_hol_wait_ms() const {
  return mean([](const TelemetrySample& s) { return s.hol_wait_ms; });
}

void Controller::observe(const TelemetrySample& s) {
  if (s.t_ms < last_obs_) throw std::logic_error("controller: out-of-order telemetry event");
  last_obs_ = s.t_ms;
  window_.push(s);
}

// reference controller.cpp:86-150: pressure -> SWAP_NEXT(min(step, cap - depth));
// sustained low usage -> DETACH(attach record) + RESTORE_NEXT(1), hysteresis both ways.
DecideOutcome Controller::decide(double now, const MorphView& view) {
  DecideOutcome out;
  if (!cfg_.enabled) return out;
  const double kv = window_.mean_kv_usage();
  const double hol = window_.mean_hol_wait_ms();
  const bool kv_hot = kv > cfg_.kv_trigger;
  if (kv_hot || hol > cfg_.queue_trigger_ms) {
    low_since_.reset();
    if (view.transaction_in_flight) return out;
    if (last_restore_ && now - *last_restore_ < cfg_.hold_ms) {
      out.notes.push_back("hysteresis_hold_after_restore");
      return out;
    }
    if (view.commanded_depth >= cfg_.max_swapped_layers) {
      ++cap_events_;
      if (!cap_noted_) {
        out.notes.push_back("swap_cap_reached");
        cap_noted_ = true;
      }
      return out;
    }
    cap_noted_ = false;
    out.commands.push_back({CommandKind::kSwapNext, std::min(cfg_.swap_step, cfg_.max_swapped_layers - view.commanded_depth), 0});
    out.notes.push_back(kv_hot ? "kv_usage_trigger" : "queue_wait_trigger");
    last_swap_ = now;
    return out;
  }
  cap_noted_ = false;
  if (!(kv < cfg_.kv_low)) {
    low_since_.reset();
    return out;
  }
  if (!low_since_) low_since_ = now;
  if (view.commanded_depth == 0 || view.transaction_in_flight) return out;
  if (now - *low_since_ < cfg_.hold_ms) return out;
  if (last_swap_ && now - *last_swap_ < cfg_.hold_ms) {
    out.notes.push_back("hysteresis_hold_after_swap");
    return out;
  }
  if (last_restore_ && now - *last_restore_ < cfg_.hold_ms) return out;
  if (view.next_restore_attached_blocks > 0)
    out.commands.push_back({CommandKind::kDetach, 0, view.next_restore_attached_blocks});
  out.commands.push_back({CommandKind::kRestoreNext, 1, 0});
  out.notes.push_back("kv_low_restore");
  last_restore_ = now;
  return out;
}

// ------------------------------------------------------------- MorphState
MorphState::MorphState(const SimModelConfig& model, Precision initial)
    : model_(model),
      tags_(static_cast<size_t>(model.num_layers), initial),
      flight_(static_cast<size_t>(model.num_layers), false),
      bytes_(static_cast<int64_t>(model.num_layers) * model.bytes(initial)) {}

double MorphState::begin_swap(int layer, Precision to, const CostModel& cost) {  // engine.cpp:19-28
  if (layer < 0 || layer >= static_cast<int>(tags_.size())) throw std::invalid_argument("begin_swap: layer out of range");
  if (flight_[layer]) throw std::invalid_argument("begin_swap: swap already in flight on layer");
  if (tags_[layer] == to) throw std::invalid_argument("begin_swap: layer already at target precision");
  flight_[layer] = true;
  ++n_flight_;
  return cost.swap_duration_ms(model_.bytes(to));
}

int64_t MorphState::complete_swap(int layer, Precision to) {  // engine.cpp:30-38
  if (!flight_[layer]) throw std::logic_error("complete_swap: no swap in flight on layer");
  flight_[layer] = false;
  --n_flight_;
  const int64_t delta = model_.bytes(to) - model_.bytes(tags_[layer]);
  tags_[layer] = to;
  bytes_ += delta;
  return delta;
}

int MorphState::quantized_count() const {
  return static_cast<int>(std::count_if(tags_.begin(), tags_.end(), [](Precision p) { return p != Precision::kFull; }));
}

SwapSequence front_to_back_sequence(int num_layers) {
  SwapSequence s;
  s.order.resize(static_cast<size_t>(num_layers));
  std::iota(s.order.begin(), s.order.end(), 0);
  return s;
}

// ------------------------------------------------------------------ traces
namespace {
int64_t round_half_up(double x) { return static_cast<int64_t>(std::floor(x + 0.5)); }

// The reference's Rng (random.hpp:13-50): mt19937_64 raw draws, hand-rolled
// conversions, so synthetic traces are identical to the reference's.
struct Rng64 {
  explicit Rng64(uint64_t seed) : g(seed) {}
  std::mt19937_64 g;
  uint64_t u64() { return g(); }
  double unit() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
  double expo() { return -std::log1p(-unit()); }
};
}  // namespace

Trace parse_trace_text(const std::string& text, const std::string& label) {  // reference trace.cpp:25-62
  Trace t;
  t.source_label = label;
  std::istringstream in(text);
  std::string line;
  int no = 0;
  auto bad = [&](const std::string& why) {
    throw std::runtime_error(label + ":" + std::to_string(no) + ": " + why);
  };
  while (std::getline(in, line)) {
    ++no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    const size_t first = line.find_first_not_of(" \t");
    if (first == std::string::npos || line[first] == '#') continue;
    TraceEvent ev;
    char c1 = 0, c2 = 0;
    std::istringstream f(line);
    if (!(f >> ev.arrival_ms >> c1 >> ev.prompt_tokens >> c2 >> ev.output_tokens) || c1 != ',' || c2 != ',')
      bad("expected `arrival_ms,prompt_tokens,output_tokens`, got `" + line + "`");
    std::string rest;
    if (f >> rest) bad("trailing data `" + rest + "`");
    if (ev.arrival_ms < 0) bad("negative arrival_ms");
    if (ev.prompt_tokens < 1) bad("prompt_tokens must be >= 1");
    if (ev.output_tokens < 1) bad("output_tokens must be >= 1");
    t.events.push_back(ev);
  }
  auto earlier = [](const TraceEvent& a, const TraceEvent& b) { return a.arrival_ms < b.arrival_ms; };
  if (!std::is_sorted(t.events.begin(), t.events.end(), earlier)) {
    std::stable_sort(t.events.begin(), t.events.end(), earlier);
    t.reordered_on_load = true;
  }
  return t;
}

Trace parse_trace(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open trace file: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return parse_trace_text(ss.str(), path);
}

std::string serialize_trace(const Trace& t) {
  std::string out = "# arrival_ms,prompt_tokens,output_tokens\n";
  for (const auto& e : t.events)
    out += std::to_string(e.arrival_ms) + "," + std::to_string(e.prompt_tokens) + "," +
           std::to_string(e.output_tokens) + "\n";
  return out;
}
void serialize_trace(const Trace& t, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write trace file: " + path);
  out << serialize_trace(t);
}

Trace downscale(const Trace& t, double factor) {  // reference trace.cpp:83-95
  if (!(factor > 0.0)) throw std::invalid_argument("downscale factor must be > 0");
  Trace out = t;
  if (out.events.empty()) return out;
  const int64_t first = t.events.front().arrival_ms;
  for (size_t i = 0; i < out.events.size(); ++i)
    out.events[i].arrival_ms = first + round_half_up(static_cast<double>(t.events[i].arrival_ms - first) * factor);
  return out;
}

Trace synth_burst(const BurstSpec& s) {  // reference trace.cpp:97-150
  if (!(s.base_rps > 0.0) || !(s.burst_rps > 0.0)) throw std::invalid_argument("synth_burst: rates must be > 0");
  if (s.total_ms < 0 || s.burst_len_ms < 0 || s.burst_start_ms < 0 || s.burst_start_ms + s.burst_len_ms > s.total_ms)
    throw std::invalid_argument("synth_burst: burst window must lie inside [0, total_ms]");
  if (s.prompt_tokens < 1 || s.output_tokens < 1) throw std::invalid_argument("synth_burst: token counts must be >= 1");
  Trace t;
  t.source_label = "synth";
  if (s.total_ms == 0) return t;
  Rng64 rng(s.seed);
  const double b0 = static_cast<double>(s.burst_start_ms);
  const double b1 = static_cast<double>(s.burst_start_ms + s.burst_len_ms);
  const double end = static_cast<double>(s.total_ms);
  double now = 0.0;
  double left = rng.expo();  // exponential "work" carried across rate changes
  while (now < end) {
    const double rate = ((now >= b0 && now < b1) ? s.burst_rps : s.base_rps) / 1000.0;
    const double edge = now < b0 ? b0 : (now < b1 ? b1 : end);
    const double avail = (edge - now) * rate;
    if (left > avail) {
      left -= avail;
      now = edge;
      continue;
    }
    now += left / rate;
    if (now >= end) break;
    t.events.push_back({round_half_up(now), s.prompt_tokens, s.output_tokens});
    left = rng.expo();
  }
  return t;
}

// Gamma(k, theta) inter-arrivals by Marsaglia-Tsang (k >= 1) with the
// k < 1 boost G(k) = G(k+1) * U^(1/k); mean gap = 1000/rps ms.
Trace synth_gamma(uint64_t seed, double rps, double shape, int64_t total_ms, int prompt, int output) {
  if (!(rps > 0.0) || !(shape > 0.0) || total_ms < 0) throw std::invalid_argument("synth_gamma: bad parameters");
  Rng64 rng(seed);
  auto normal = [&]() {
    double u1 = rng.unit(), u2 = rng.unit();
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  };
  auto gamma1 = [&](double k) {  // k >= 1, unit scale
    const double d = k - 1.0 / 3.0, c = 1.0 / std::sqrt(9.0 * d);
    for (;;) {
      double x = normal(), v = 1.0 + c * x;
      if (v <= 0.0) continue;
      v = v * v * v;
      const double u = rng.unit();
      if (u < 1.0 - 0.0331 * x * x * x * x) return d * v;
      if (std::log(std::max(u, 1e-300)) < 0.5 * x * x + d * (1.0 - v + std::log(v))) return d * v;
    }
  };
  const double theta = (1000.0 / rps) / shape;
  Trace t;
  t.source_label = "gamma";
  double now = 0.0;
  for (;;) {
    double g = shape >= 1.0 ? gamma1(shape) : gamma1(shape + 1.0) * std::pow(std::max(rng.unit(), 1e-300), 1.0 / shape);
    now += g * theta;
    if (now >= static_cast<double>(total_ms)) break;
    t.events.push_back({round_half_up(now), prompt, output});
  }
  return t;
}

// ----------------------------------------------------------------- metrics
std::optional<double> percentile_nearest_rank(std::vector<double> v, double p) {  // metrics.cpp:12-18
  if (v.empty()) return std::nullopt;
  if (p <= 0.0 || p > 100.0) throw std::invalid_argument("percentile must be in (0, 100]");
  std::sort(v.begin(), v.end());
  const size_t rank = static_cast<size_t>(std::ceil(p / 100.0 * static_cast<double>(v.size())));
  return v[std::max<size_t>(rank, 1) - 1];
}

PercentileSummary PercentileSummary::of(const std::vector<double>& v) {
  PercentileSummary s;
  s.count = static_cast<int64_t>(v.size());
  if (v.empty()) return s;
  s.p50 = percentile_nearest_rank(v, 50.0);
  s.p95 = percentile_nearest_rank(v, 95.0);
  s.p99 = percentile_nearest_rank(v, 99.0);
  s.mean = std::accumulate(v.begin(), v.end(), 0.0) / static_cast<double>(v.size());
  s.max = *std::max_element(v.begin(), v.end());
  return s;
}

void StepSeries::record(double t, double v) {  // right-continuous steps, metrics.cpp:46-53
  if (!points.empty() && points.back().first == t) {
    points.back().second = v;
    return;
  }
  if (!points.empty() && points.back().second == v) return;
  points.emplace_back(t, v);
}
double StepSeries::at(double t) const {
  double v = 0.0;
  for (const auto& p : points) {
    if (p.first > t) break;
    v = p.second;
  }
  return v;
}
double StepSeries::peak() const {
  double best = 0.0;
  for (const auto& p : points) best = std::max(best, p.second);
  return best;
}
double StepSeries::time_weighted_mean(double t_end) const {  // metrics.cpp:70-81
  if (points.empty() || t_end <= points.front().first) return 0.0;
  double acc = 0.0;
  for (size_t i = 0; i < points.size(); ++i) {
    const double t0 = points[i].first;
    if (t0 >= t_end) break;
    const double t1 = i + 1 < points.size() ? std::min(points[i + 1].first, t_end) : t_end;
    if (t1 > t0) acc += points[i].second * (t1 - t0);
  }
  const double span = t_end - points.front().first;
  return span > 0.0 ? acc / span : 0.0;
}
std::string Timelines::to_csv(double t_end_ms) const {
  std::string out = "t_ms,kv_capacity_blocks,kv_used_blocks,quantized_layers,queue_depth\n";
  char buf[160];
  const int64_t last = static_cast<int64_t>(std::ceil(t_end_ms / 1000.0)) * 1000;
  for (int64_t t = 0; t <= last; t += 1000) {
    const double td = static_cast<double>(t);
    std::snprintf(buf, sizeof(buf), "%lld,%lld,%lld,%lld,%lld\n", static_cast<long long>(t),
                  static_cast<long long>(kv_capacity_blocks.at(td)), static_cast<long long>(kv_used_blocks.at(td)),
                  static_cast<long long>(quantized_layers.at(td)), static_cast<long long>(queue_depth.at(td)));
    out += buf;
  }
  return out;
}

std::string EventLog::to_text() const {
  std::string out;
  char prefix[64];
  for (const auto& e : entries) {
    std::snprintf(prefix, sizeof(prefix), "%llu %.6f ", static_cast<unsigned long long>(e.seq), e.t_ms);
    out += prefix;
    out += e.text;
    out += '\n';
  }
  return out;
}

namespace {
std::string jnum(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}
std::string jopt(const std::optional<double>& v) { return v ? jnum(*v) : "null"; }
std::string jsum(const PercentileSummary& s) {
  return "{\"count\":" + std::to_string(s.count) + ",\"max\":" + jopt(s.max) + ",\"mean\":" + jopt(s.mean) +
         ",\"p50\":" + jopt(s.p50) + ",\"p95\":" + jopt(s.p95) + ",\"p99\":" + jopt(s.p99) + "}";
}
std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o + "\"";
}
}  // namespace

// Same schema as the reference report (metrics.cpp:98-144) plus a "device" block.
std::string MetricsReport::to_json() const {
  std::string j = "{";
  j += "\"arm\":" + jstr(arm) + ",\"fingerprint\":" + jstr(fingerprint) + ",\"seed\":" + std::to_string(seed);
  j += ",\"slo_ms\":" + jnum(slo_ms);
  j += ",\"requests\":{\"completed\":" + std::to_string(completed_requests) +
       ",\"preemptions\":" + std::to_string(preemption_count) + ",\"total\":" + std::to_string(total_requests) +
       ",\"unserviceable\":" + std::to_string(unserviceable_requests) + "}";
  j += ",\"ttft_ms\":" + jsum(ttft_ms) + ",\"tpot_ms\":" + jsum(tpot_ms) + ",\"e2e_ms\":" + jsum(e2e_ms) +
       ",\"queue_ms\":" + jsum(queue_ms);
  j += ",\"slo\":{\"rate\":" + jnum(slo_violation_rate) + ",\"violations\":" + std::to_string(slo_violations) + "}";
  j += ",\"throughput_rps\":" + jnum(throughput_rps) + ",\"sim_end_ms\":" + jnum(sim_end_ms);
  j += ",\"kv\":{\"mean_utilization\":" + jnum(kv_mean_utilization) +
       ",\"peak_capacity_blocks\":" + std::to_string(kv_peak_capacity_blocks) +
       ",\"peak_used_blocks\":" + std::to_string(kv_peak_used_blocks) +
       ",\"static_capacity_blocks\":" + std::to_string(kv_static_capacity_blocks) + "}";
  j += ",\"morph\":{\"peak_quantized_layers\":" + std::to_string(peak_quantized_layers) +
       ",\"restore_events\":" + std::to_string(restore_events) +
       ",\"saturation_cap_events\":" + std::to_string(saturation_cap_events) +
       ",\"swap_events\":" + std::to_string(swap_events) + "}";
  j += ",\"exposure\":{\"fraction\":" + jnum(exposure_fraction) +
       ",\"token_layer_quant_sum\":" + std::to_string(token_layer_quant_sum) +
       ",\"tokens_quantized\":" + std::to_string(tokens_quantized) + ",\"tokens_total\":" + std::to_string(tokens_total) +
       "}";
  j += ",\"per_request\":[";
  for (size_t i = 0; i < per_request.size(); ++i) {
    const auto& r = per_request[i];
    if (i) j += ",";
    j += "{\"arrival_ms\":" + std::to_string(r.arrival_ms) + ",\"e2e_ms\":" + jnum(r.e2e_ms) +
         ",\"id\":" + std::to_string(r.id) + ",\"output_tokens\":" + std::to_string(r.output_tokens) +
         ",\"preemptions\":" + std::to_string(r.preemptions) + ",\"prompt_tokens\":" + std::to_string(r.prompt_tokens) +
         ",\"queue_ms\":" + jnum(r.queue_ms) + ",\"token_layer_quant_sum\":" + std::to_string(r.token_layer_quant_sum) +
         ",\"tokens_quantized\":" + std::to_string(r.tokens_quantized) + ",\"tpot_ms\":" + jopt(r.tpot_ms) +
         ",\"ttft_ms\":" + jnum(r.ttft_ms) + "}";
  }
  j += "]";
  j += ",\"device\":{\"busy_ms\":" + jnum(device_busy_ms) + ",\"decode_ms\":" + jnum(decode_ms) +
       ",\"decode_steps\":" + std::to_string(decode_steps) + ",\"decode_tokens\":" + jnum(decode_tokens) +
       ",\"exposed_swap_stall_ms\":" + jnum(exposed_swap_stall_ms) + ",\"prefill_ms\":" + jnum(prefill_ms) +
       ",\"prefill_tokens\":" + std::to_string(prefill_tokens) + ",\"swap_upload_ms\":" + jnum(swap_upload_ms) +
       ",\"decode_steps_overlap\":" + std::to_string(decode_steps_overlap) +
       ",\"decode_ms_overlap\":" + jnum(decode_ms_overlap) +
       ",\"exposed_stall_ms_per_token\":" + jnum(exposed_stall_ms_per_token) +
       ",\"host_gap_ms\":" + jnum(host_gap_ms) + ",\"graph_captures\":" + std::to_string(graph_captures) + "}";
  j += "}";
  return j;
}

}  // namespace morphserve
