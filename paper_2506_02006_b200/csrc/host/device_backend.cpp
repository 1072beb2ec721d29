// device_backend.cpp -- DeviceBackend over the C ABI (include/morphserve.h).
// The engine's request id is the device token-history slot; prompts are
// synthetic token ids drawn from a counter RNG so CPU and GPU runs see the
// same inputs.
#include "device_backend.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>

namespace morphserve {

namespace {
void ck(int rc, const char* what) {
  if (rc == MS_OK) return;
  const std::string msg = std::string(what) + ": " + ms_last_error();
  if (rc == MS_EVALIDATION) throw std::invalid_argument(msg);
  if (rc == MS_ELOGIC) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}
uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
}  // namespace

std::vector<int32_t> synthetic_prompt(uint64_t seed, int req, int n, int vocab) {
  std::vector<int32_t> t(static_cast<size_t>(n));
  const uint64_t key = mix(seed ^ (0xA24BAED4963EE407ull * (uint64_t)(req + 1)));
  for (int i = 0; i < n; ++i) t[i] = static_cast<int32_t>(mix(key + (uint64_t)i) % (uint64_t)vocab);
  return t;
}

CAbiBackend::CAbiBackend(ms_ctx* ctx, int vocab, bool measure) : ctx_(ctx), vocab_(vocab), measure_(measure) {
  if (!ctx_) throw std::invalid_argument("device backend: null context");
}

void CAbiBackend::on_run_start(const std::vector<TraceEvent>& reqs, uint64_t seed) {
  ck(ms_reset_state(ctx_), "ms_reset_state");  // every run starts all-BF16 with no KV mapped
  int max_len = 2;
  for (const auto& r : reqs) max_len = std::max(max_len, r.prompt_tokens + r.output_tokens + 1);
  ck(ms_hist_reserve(ctx_, std::max<int>(1, (int)reqs.size()), max_len), "ms_hist_reserve");
  for (size_t i = 0; i < reqs.size(); ++i) {
    const auto p = synthetic_prompt(seed, (int)i, reqs[i].prompt_tokens, vocab_);
    ck(ms_hist_write(ctx_, (int32_t)i, 0, p.data(), (int32_t)p.size()), "ms_hist_write");
  }
}

void CAbiBackend::record(char kind, std::vector<int> reqs, std::vector<int> pos) {
  if (!record_) return;
  DeviceCall c{kind, std::move(reqs), std::move(pos), {}};
  for (int l = 0; l < layers_; ++l) c.bits.push_back(ms_layer_bits(ctx_, l));
  calls_.push_back(std::move(c));
}

double CAbiBackend::prefill(int req, int tokens, const std::vector<BlockId>& blocks) {
  record('P', {req}, {tokens});
  ck(ms_prefill(ctx_, req, tokens, blocks.data(), (int32_t)blocks.size(), nullptr, nullptr), "ms_prefill");
  return measured();
}

double CAbiBackend::decode(const std::vector<Row>& rows) {
  const int n = (int)rows.size();
  size_t width = 1;
  for (const auto& r : rows) width = std::max(width, r.blocks->size());
  slots_.resize(n);
  pos_.resize(n);
  table_.assign((size_t)n * width, -1);
  for (int i = 0; i < n; ++i) {
    slots_[i] = rows[i].req;
    pos_[i] = rows[i].pos;
    std::copy(rows[i].blocks->begin(), rows[i].blocks->end(), table_.begin() + (size_t)i * width);
  }
  record('D', std::vector<int>(slots_.begin(), slots_.end()), std::vector<int>(pos_.begin(), pos_.end()));
  ms_decode_batch b{n, slots_.data(), pos_.data(), nullptr, table_.data(), (int32_t)width};
  ck(ms_decode_step(ctx_, &b, nullptr, nullptr), "ms_decode_step");
  return measured();
}

double CAbiBackend::measured() {
  if (!measure_) return 0.0;
  float ms = 0.f;
  ck(ms_last_step_ms(ctx_, &ms), "ms_last_step_ms");
  return ms;
}

void CAbiBackend::swap_begin(int layer, int bits) {
  uint64_t t = 0;
  ck(ms_swap_begin(ctx_, layer, bits, &t), "ms_swap_begin");
  tickets_[layer] = t;
}

bool CAbiBackend::swap_ready(int layer, double* upload_ms) {
  auto it = tickets_.find(layer);
  if (it == tickets_.end()) throw std::logic_error("swap_ready: no swap in flight");
  int done = 0;
  ck(ms_swap_poll(ctx_, it->second, &done), "ms_swap_poll");
  if (done && upload_ms) {
    float ms = 0.f;
    ck(ms_swap_wait(ctx_, it->second, &ms), "ms_swap_wait");
    *upload_ms = ms;
  }
  return done != 0;
}

double CAbiBackend::swap_wait(int layer) {
  auto it = tickets_.find(layer);
  if (it == tickets_.end()) throw std::logic_error("swap_wait: no swap in flight");
  float ms = 0.f;
  ck(ms_swap_wait(ctx_, it->second, &ms), "ms_swap_wait");
  return ms;
}

int64_t CAbiBackend::graph_captures() { return ms_graph_captures(ctx_); }

void CAbiBackend::swap_commit(int layer, double* upload_ms) {
  auto it = tickets_.find(layer);
  if (it == tickets_.end()) throw std::logic_error("swap_commit: no swap in flight");
  if (upload_ms) {
    *upload_ms = 0.0;
    int done = 0;
    ck(ms_swap_poll(ctx_, it->second, &done), "ms_swap_poll");
    if (done) {
      float ms = 0.f;
      ck(ms_swap_wait(ctx_, it->second, &ms), "ms_swap_wait");
      *upload_ms = ms;
    }
  }
  int64_t freed = 0;
  ck(ms_swap_commit(ctx_, it->second, &freed), "ms_swap_commit");
  tickets_.erase(it);
}

void CAbiBackend::kv_attach(BlockId first_id, int64_t n) { ck(ms_kv_attach(ctx_, first_id, n), "ms_kv_attach"); }

void CAbiBackend::kv_detach(const std::vector<BlockId>& ids) {
  ck(ms_kv_detach(ctx_, ids.data(), (int64_t)ids.size()), "ms_kv_detach");
}

void CAbiBackend::finish() { ck(ms_sync(ctx_), "ms_sync"); }

}  // namespace morphserve
