// device_backend.hpp -- the engine's DeviceBackend bound to libmorphserve.so.
#pragma once

#include <map>
#include <vector>

#include "../../../include/morphserve.h"
#include "host.hpp"

namespace morphserve {

std::vector<int32_t> synthetic_prompt(uint64_t seed, int req, int n, int vocab);

// One executed device call, for replay against the CPU oracle.
struct DeviceCall {
  char kind;                        // 'P' prefill, 'D' decode
  std::vector<int> reqs, pos;       // prefill: pos = token count
  std::vector<int> bits;            // committed precision of every layer at launch
};

class CAbiBackend final : public DeviceBackend {
 public:
  // measure = true: every step is timed with CUDA events (ClockMode::kDevice).
  CAbiBackend(ms_ctx* ctx, int vocab, bool measure);
  void on_run_start(const std::vector<TraceEvent>& reqs, uint64_t seed) override;
  double prefill(int req, int tokens, const std::vector<BlockId>& blocks) override;
  double decode(const std::vector<Row>& rows) override;
  void swap_begin(int layer, int bits) override;
  void swap_commit(int layer, double* upload_ms) override;
  bool swap_ready(int layer, double* upload_ms) override;
  double swap_wait(int layer) override;
  int64_t graph_captures() override;
  void kv_attach(BlockId first_id, int64_t n) override;
  void kv_detach(const std::vector<BlockId>& ids) override;
  void finish() override;
  void set_recording(bool on, int num_layers) {
    record_ = on;
    layers_ = num_layers;
  }
  const std::vector<DeviceCall>& calls() const { return calls_; }

 private:
  void record(char kind, std::vector<int> reqs, std::vector<int> pos);
  bool record_ = false;
  int layers_ = 0;
  std::vector<DeviceCall> calls_;
  double measured();
  ms_ctx* ctx_;
  int vocab_;
  bool measure_;
  std::map<int, uint64_t> tickets_;
  std::vector<int32_t> slots_, pos_;
  std::vector<int64_t> table_;
};

}  // namespace morphserve
