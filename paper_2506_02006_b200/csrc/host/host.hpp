// host.hpp -- C++ host runtime of the B200 serving path.
//
// Same public types and semantics as the reference simulator's headers
// (proj/include/morphsim/{kv_pool,controller,engine,sim_config,metrics,trace}.hpp)
// so the engine, LayerSwapper state and KV resizer stay drop-in; the
// difference is the DeviceBackend seam: every prefill, decode step, layer swap
// and KV attach/detach the event loop schedules is also executed on the B200
// through include/morphserve.h.  Two clock modes:
//   kVirtual -- durations from CostModel (reference arithmetic, sim_config.cpp:23-33),
//               so the event log / block tables are bit-identical to the reference;
//   kDevice  -- durations measured on the GPU (CUDA events), so TTFT/TPOT are real.
#pragma once

#include <array>
#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <optional>
#include <string>
#include <vector>

namespace morphserve {

// ------------------------------------------------------------ precision tags
enum class Precision { kFull = 0, kQ8 = 1, kQ4 = 2, kQ3 = 3 };  // reference toy_model.hpp:26
int precision_bits(Precision p);
Precision precision_from_bits(int bits);
std::string precision_name(Precision p);

// ------------------------------------------------------------ cost model
constexpr int64_t kGiB = 1024LL * 1024 * 1024;
constexpr int64_t kMiB = 1024LL * 1024;
int64_t gib_to_bytes(double gib);

struct SimModelConfig {  // reference sim_config.hpp:17-28
  int num_layers = 32;
  std::array<int64_t, 4> layer_bytes = {gib_to_bytes(0.4), gib_to_bytes(0.2), gib_to_bytes(0.1),
                                        gib_to_bytes(0.075)};
  int64_t bytes(Precision p) const { return layer_bytes[static_cast<int>(p)]; }
  int64_t model_bytes_at(Precision p) const { return static_cast<int64_t>(num_layers) * bytes(p); }
  void validate() const;
};

struct CostModel {  // reference sim_config.hpp:31-45
  double prefill_ms_per_token = 0.02;
  std::array<double, 4> decode_ms_per_layer = {0.3, 0.24, 0.18, 0.15};
  double attn_ms_per_kv_block = 0.00005;
  double pcie_gib_per_s = 26.0;
  double swap_fixed_overhead_ms = 2.0;
  int64_t max_batch_tokens = 100000;
  double decode_step_ms(const std::vector<Precision>& tags, int64_t batch_blocks) const;
  double swap_duration_ms(int64_t variant_bytes) const;
  void validate() const;
};

struct MemoryBudget {
  int64_t device_bytes = 24 * kGiB;
  int64_t reserve_bytes = 4 * kGiB;
};

// ------------------------------------------------------------ KV block pool
using RequestId = int;
using BlockId = int64_t;

struct KvConfig {  // reference kv_pool.hpp:14-18
  int block_tokens = 16;
  int64_t block_bytes = 2 * 1024 * 1024;
  int64_t static_capacity_blocks = 0;
};

struct DetachResult {
  int64_t removed_now = 0;
  int64_t deferred = 0;
  int64_t capacity_blocks = 0;
};

// Elastic paged block pool (semantics of reference kv_pool.cpp:9-158).
// Every id that leaves the pool (immediate or deferred detach) is also queued
// in `retired()` so the device backend can return its arena page.
class KvBlockPool {
 public:
  explicit KvBlockPool(const KvConfig& config);
  void admit(RequestId req);
  bool is_admitted(RequestId req) const { return reqs_.count(req) > 0; }
  std::optional<std::vector<BlockId>> alloc_for_tokens(RequestId req, int64_t new_tokens);
  int64_t release(RequestId req);
  int64_t attach_blocks(int64_t n);
  DetachResult detach_blocks(int64_t n);
  std::optional<RequestId> preempt_victim(const std::function<bool(RequestId)>& eligible);

  int64_t capacity_blocks() const { return capacity_; }
  int64_t free_blocks() const { return static_cast<int64_t>(free_.size()); }
  int64_t used_blocks() const { return capacity_ - free_blocks(); }
  int64_t attached_extra_blocks() const { return attached_; }
  int64_t pending_detach_blocks() const { return pending_detach_; }
  int64_t tokens_of(RequestId req) const;
  int64_t blocks_of(RequestId req) const;
  const std::vector<BlockId>& block_list(RequestId req) const;
  double usage_fraction() const;
  const KvConfig& config() const { return cfg_; }
  BlockId next_block_id() const { return next_id_; }
  std::vector<BlockId> take_retired();
  void check_invariants() const;
  int64_t blocks_needed_for(int64_t existing_tokens, int64_t new_tokens) const;

 private:
  struct Entry {
    int64_t tokens = 0;
    std::vector<BlockId> blocks;
    uint64_t stamp = 0;
  };
  void drain_pending_detach();

  KvConfig cfg_;
  int64_t capacity_ = 0, attached_ = 0, pending_detach_ = 0;
  BlockId next_id_ = 0;
  uint64_t next_stamp_ = 0;
  std::vector<BlockId> free_;  // LIFO stack: back() is the top
  std::map<RequestId, Entry> reqs_;
  std::vector<BlockId> retired_;
};

// ------------------------------------------------------------ controller
enum class ControllerMode { kAccuracy, kPerformance };

struct ControllerConfig {  // reference controller.hpp:16-30
  bool enabled = false;
  ControllerMode mode = ControllerMode::kPerformance;
  double kv_trigger = 0.85;
  double kv_low = 0.70;
  double queue_trigger_ms = 100;
  double hold_ms = 500;
  int max_swapped_layers = 1;
  int swap_step = 1;
  double telemetry_window_ms = 200;
  int target_bits = 4;
  void validate(int num_layers) const;
  static ControllerConfig defaults_for(ControllerMode mode, int num_layers);
};

struct TelemetrySample {
  double t_ms = 0.0, kv_usage = 0.0, queue_depth = 0.0, hol_wait_ms = 0.0;
};

class TelemetryWindow {
 public:
  explicit TelemetryWindow(double window_ms) : window_ms_(window_ms) {}
  void push(const TelemetrySample& s);
  double mean_kv_usage() const;
  double mean_queue_depth() const;
  double mean_hol_wait_ms() const;

 private:
  template <class Get>
  double mean(Get get) const;
  double window_ms_;
  std::deque<TelemetrySample> samples_;
  TelemetrySample last_;
};

enum class CommandKind { kSwapNext, kRestoreNext, kAttach, kDetach };
struct Command {
  CommandKind kind;
  int count = 0;
  int64_t blocks = 0;
};
struct MorphView {
  int num_layers = 0;
  int commanded_depth = 0;
  bool transaction_in_flight = false;
  int64_t next_restore_attached_blocks = 0;
};
struct DecideOutcome {
  std::vector<Command> commands;
  std::vector<std::string> notes;
};

class Controller {  // decision logic of reference controller.cpp:86-150
 public:
  explicit Controller(const ControllerConfig& cfg) : cfg_(cfg), window_(cfg.telemetry_window_ms) {}
  void observe(const TelemetrySample& s);
  DecideOutcome decide(double now_ms, const MorphView& view);
  int64_t saturation_cap_events() const { return cap_events_; }
  const ControllerConfig& config() const { return cfg_; }

 private:
  ControllerConfig cfg_;
  TelemetryWindow window_;
  double last_obs_ = -1.0;
  std::optional<double> low_since_, last_swap_, last_restore_;
  int64_t cap_events_ = 0;
  bool cap_noted_ = false;
};

// ------------------------------------------------------------ LayerSwapper state
class MorphState {  // reference engine.hpp:22-45
 public:
  MorphState(const SimModelConfig& model, Precision initial);
  double begin_swap(int layer, Precision to, const CostModel& cost);
  int64_t complete_swap(int layer, Precision to);
  bool swap_in_flight(int layer) const { return flight_[layer]; }
  int in_flight_count() const { return n_flight_; }
  Precision tag(int layer) const { return tags_[layer]; }
  const std::vector<Precision>& tags() const { return tags_; }
  int quantized_count() const;
  int64_t model_bytes() const { return bytes_; }

 private:
  SimModelConfig model_;
  std::vector<Precision> tags_;
  std::vector<bool> flight_;
  int n_flight_ = 0;
  int64_t bytes_ = 0;
};

// ------------------------------------------------------------ traces
struct TraceEvent {
  int64_t arrival_ms = 0;
  int prompt_tokens = 0;
  int output_tokens = 0;
  bool operator==(const TraceEvent&) const = default;
};
struct Trace {
  std::vector<TraceEvent> events;
  std::string source_label;
  bool reordered_on_load = false;
};
Trace parse_trace_text(const std::string& text, const std::string& label);
Trace parse_trace(const std::string& path);
std::string serialize_trace(const Trace& t);
void serialize_trace(const Trace& t, const std::string& path);
Trace downscale(const Trace& t, double factor);
struct BurstSpec {
  uint64_t seed = 0;
  double base_rps = 1.0, burst_rps = 1.0;
  int64_t burst_start_ms = 0, burst_len_ms = 0, total_ms = 0;
  int prompt_tokens = 1, output_tokens = 1;
};
Trace synth_burst(const BurstSpec& spec);
// Gamma-renewal arrivals (shape k, mean rate rps): CV = 1/sqrt(k); k = 0.25 is
// the paper's bursty setting (BASELINE.json config 3).  Not in the reference.
Trace synth_gamma(uint64_t seed, double rps, double shape, int64_t total_ms, int prompt_tokens, int output_tokens);

// ------------------------------------------------------------ metrics
std::optional<double> percentile_nearest_rank(std::vector<double> values, double p);
struct PercentileSummary {
  std::optional<double> p50, p95, p99, mean, max;
  int64_t count = 0;
  static PercentileSummary of(const std::vector<double>& v);
};
struct StepSeries {
  std::vector<std::pair<double, double>> points;
  void record(double t, double v);
  double at(double t) const;
  double peak() const;
  double time_weighted_mean(double t_end) const;
};
struct Timelines {
  StepSeries kv_capacity_blocks, kv_used_blocks, quantized_layers, queue_depth;
  std::string to_csv(double t_end_ms) const;
};
struct PerRequestMetrics {
  int id = 0;
  int64_t arrival_ms = 0;
  int prompt_tokens = 0, output_tokens = 0;
  double ttft_ms = 0.0;
  std::optional<double> tpot_ms;
  double e2e_ms = 0.0, queue_ms = 0.0;
  int preemptions = 0;
  int64_t tokens_quantized = 0, token_layer_quant_sum = 0;
};
struct MetricsReport {
  std::string arm, fingerprint;
  uint64_t seed = 0;
  double slo_ms = 0.0;
  int64_t total_requests = 0, completed_requests = 0, unserviceable_requests = 0, preemption_count = 0;
  PercentileSummary ttft_ms, tpot_ms, e2e_ms, queue_ms;
  int64_t slo_violations = 0;
  double slo_violation_rate = 0.0, throughput_rps = 0.0, sim_end_ms = 0.0;
  int64_t kv_static_capacity_blocks = 0, kv_peak_capacity_blocks = 0, kv_peak_used_blocks = 0;
  double kv_mean_utilization = 0.0;
  int64_t swap_events = 0, restore_events = 0, peak_quantized_layers = 0, saturation_cap_events = 0;
  int64_t tokens_total = 0, tokens_quantized = 0, token_layer_quant_sum = 0;
  double exposure_fraction = 0.0;
  std::vector<PerRequestMetrics> per_request;
  // device-side additions (kDevice clock / device-backed runs)
  double device_busy_ms = 0.0, decode_ms = 0.0, prefill_ms = 0.0, decode_tokens = 0.0;
  int64_t decode_steps = 0, prefill_tokens = 0;
  double swap_upload_ms = 0.0, exposed_swap_stall_ms = 0.0;
  // kWall: decode steps that overlapped an in-flight upload, their time above
  // the no-upload step-time model (least squares over the other steps:
  // ms = a + b * kv_blocks + c * batch), host time between device steps
  int64_t decode_steps_overlap = 0, graph_captures = 0;
  double decode_ms_overlap = 0.0, exposed_stall_ms_per_token = 0.0, host_gap_ms = 0.0;
  std::string to_json() const;
};
struct EventLog {
  struct Entry {
    uint64_t seq;
    double t_ms;
    std::string text;
  };
  std::vector<Entry> entries;
  void append(double t, const std::string& text) { entries.push_back({(uint64_t)entries.size(), t, text}); }
  std::string to_text() const;
};

// ------------------------------------------------------------ swap order
struct SwapSequence {  // reference profiler.hpp:26-37 (consumed, not produced)
  std::vector<int> order;
  int num_layers() const { return static_cast<int>(order.size()); }
};
SwapSequence front_to_back_sequence(int num_layers);

// ------------------------------------------------------------ device seam
// What the event loop executes on the GPU.  Implemented over the C ABI in
// device_backend.cpp (class CAbiBackend); a null backend keeps the pure
// reference behaviour (cost model only).
class DeviceBackend {
 public:
  virtual ~DeviceBackend() = default;
  virtual void on_run_start(const std::vector<TraceEvent>& reqs, uint64_t seed) = 0;
  // Returns measured device ms (used only in kDevice clock mode).
  virtual double prefill(int req, int tokens, const std::vector<BlockId>& blocks) = 0;
  struct Row {
    int req;
    int pos;  // position of the input token
    const std::vector<BlockId>* blocks;
  };
  virtual double decode(const std::vector<Row>& rows) = 0;
  virtual void swap_begin(int layer, int bits) = 0;
  // Commit at a token boundary; returns freed pages.  In kDevice mode *done_ms
  // receives the measured upload time.
  virtual void swap_commit(int layer, double* upload_ms) = 0;
  virtual bool swap_ready(int layer, double* upload_ms) = 0;
  // Blocks (no spin) until the layer's upload has landed; returns its upload ms.
  virtual double swap_wait(int layer) = 0;
  // CUDA-graph captures made so far (graph-safe swaps: commits must not add any).
  virtual int64_t graph_captures() { return 0; }
  virtual void kv_attach(BlockId first_id, int64_t n) = 0;
  virtual void kv_detach(const std::vector<BlockId>& ids) = 0;
  virtual void finish() = 0;
};

// kVirtual: every duration from the CostModel (byte-identical reference logs).
// kDevice:  GPU-time simulation -- the clock advances by measured step times;
//           a swap lasts its measured upload (the host waits for it, blocking).
// kWall:    real clock -- events run on a steady wall clock (ms since start),
//           arrivals are released at their trace times, a step completes when
//           the GPU says so, and a swap completes at the first event boundary
//           after its upload has landed (polled, never waited on): decode keeps
//           running while the LayerSwapper's copies stream (reference
//           engine.cpp:397-402 future-dated kSwapDone).
enum class ClockMode { kVirtual, kDevice, kWall };

struct ArmSpec {
  std::string label = "static-full";
  Precision initial_precision = Precision::kFull;
  ControllerConfig controller;
  std::optional<SwapSequence> sequence;
};

struct EngineConfig {
  SimModelConfig model;
  KvConfig kv;
  CostModel cost;
  MemoryBudget budget;
  double slo_ms = 2000.0;
  double monitor_tick_ms = 100.0;
  void validate() const;
  int64_t auto_static_capacity_blocks() const;
};

struct RunResult {
  MetricsReport report;
  EventLog log;
  Timelines timelines;
};

RunResult run_simulation(const EngineConfig& config, const ArmSpec& arm, const Trace& trace, uint64_t seed,
                         DeviceBackend* device = nullptr, ClockMode clock = ClockMode::kVirtual);

}  // namespace morphserve
