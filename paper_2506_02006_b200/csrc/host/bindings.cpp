// bindings.cpp -- pybind11 module `_core`, the Python face of the host
// runtime.  Mirrors the reference module's surface (proj/bindings/py_module.cpp:85-224:
// TraceEvent/Trace/trace tools, KvConfig/KvBlockPool, JSON reports) and adds
// the device-backed engine entry point.
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "device_backend.hpp"
#include "host.hpp"

namespace py = pybind11;
using namespace morphserve;

namespace {

template <class T>
T get(const py::dict& d, const char* k, T def) {
  return d.contains(k) ? d[k].cast<T>() : def;
}

EngineConfig engine_from(const py::dict& d) {
  EngineConfig c;
  c.model.num_layers = get<int>(d, "num_layers", c.model.num_layers);
  if (d.contains("layer_bytes")) {
    auto v = d["layer_bytes"].cast<std::vector<int64_t>>();
    if (v.size() != 4) throw std::invalid_argument("layer_bytes needs 4 entries (full, q8, q4, q3)");
    for (int i = 0; i < 4; ++i) c.model.layer_bytes[i] = v[i];
  }
  c.kv.block_tokens = get<int>(d, "block_tokens", c.kv.block_tokens);
  c.kv.block_bytes = get<int64_t>(d, "block_bytes", c.kv.block_bytes);
  c.kv.static_capacity_blocks = get<int64_t>(d, "static_capacity_blocks", c.kv.static_capacity_blocks);
  c.budget.device_bytes = get<int64_t>(d, "device_bytes", c.budget.device_bytes);
  c.budget.reserve_bytes = get<int64_t>(d, "reserve_bytes", c.budget.reserve_bytes);
  c.cost.prefill_ms_per_token = get<double>(d, "prefill_ms_per_token", c.cost.prefill_ms_per_token);
  if (d.contains("decode_ms_per_layer")) {
    auto v = d["decode_ms_per_layer"].cast<std::vector<double>>();
    if (v.size() != 4) throw std::invalid_argument("decode_ms_per_layer needs 4 entries");
    for (int i = 0; i < 4; ++i) c.cost.decode_ms_per_layer[i] = v[i];
  }
  c.cost.attn_ms_per_kv_block = get<double>(d, "attn_ms_per_kv_block", c.cost.attn_ms_per_kv_block);
  c.cost.pcie_gib_per_s = get<double>(d, "pcie_gib_per_s", c.cost.pcie_gib_per_s);
  c.cost.swap_fixed_overhead_ms = get<double>(d, "swap_fixed_overhead_ms", c.cost.swap_fixed_overhead_ms);
  c.cost.max_batch_tokens = get<int64_t>(d, "max_batch_tokens", c.cost.max_batch_tokens);
  c.slo_ms = get<double>(d, "slo_ms", c.slo_ms);
  c.monitor_tick_ms = get<double>(d, "monitor_tick_ms", c.monitor_tick_ms);
  return c;
}

ControllerConfig controller_from(const py::dict& d) {
  ControllerConfig c;
  c.enabled = get<bool>(d, "enabled", true);
  c.mode = get<std::string>(d, "mode", "performance") == "accuracy" ? ControllerMode::kAccuracy
                                                                     : ControllerMode::kPerformance;
  c.kv_trigger = get<double>(d, "kv_trigger", c.kv_trigger);
  c.kv_low = get<double>(d, "kv_low", c.kv_low);
  c.queue_trigger_ms = get<double>(d, "queue_trigger_ms", c.queue_trigger_ms);
  c.hold_ms = get<double>(d, "hold_ms", c.hold_ms);
  c.max_swapped_layers = get<int>(d, "max_swapped_layers", c.max_swapped_layers);
  c.swap_step = get<int>(d, "swap_step", c.swap_step);
  c.telemetry_window_ms = get<double>(d, "telemetry_window_ms", c.telemetry_window_ms);
  c.target_bits = get<int>(d, "target_bits", c.target_bits);
  return c;
}

ArmSpec arm_from(const py::dict& d) {
  ArmSpec a;
  a.label = get<std::string>(d, "label", a.label);
  a.initial_precision = precision_from_bits(get<int>(d, "initial_bits", 16));
  if (d.contains("controller") && !d["controller"].is_none()) a.controller = controller_from(d["controller"].cast<py::dict>());
  if (d.contains("sequence") && !d["sequence"].is_none()) {
    SwapSequence s;
    s.order = d["sequence"].cast<std::vector<int>>();
    a.sequence = s;
  }
  return a;
}

py::dict result_dict(const RunResult& r) {
  py::dict out;
  out["report_json"] = r.report.to_json();
  out["log"] = r.log.to_text();
  out["timeline_csv"] = r.timelines.to_csv(r.report.sim_end_ms);
  return out;
}

}  // namespace

PYBIND11_MODULE(_core, m) {
  m.doc() = "B200 serving host runtime: traces, paged KV pool, controller, device-backed engine";

  py::class_<TraceEvent>(m, "TraceEvent")
      .def(py::init<>())
      .def(py::init([](int64_t a, int p, int o) { return TraceEvent{a, p, o}; }), py::arg("arrival_ms"),
           py::arg("prompt_tokens"), py::arg("output_tokens"))
      .def_readwrite("arrival_ms", &TraceEvent::arrival_ms)
      .def_readwrite("prompt_tokens", &TraceEvent::prompt_tokens)
      .def_readwrite("output_tokens", &TraceEvent::output_tokens)
      .def("__eq__", [](const TraceEvent& a, const TraceEvent& b) { return a == b; })
      .def("__repr__", [](const TraceEvent& e) {
        return "TraceEvent(" + std::to_string(e.arrival_ms) + ", " + std::to_string(e.prompt_tokens) + ", " +
               std::to_string(e.output_tokens) + ")";
      });
  py::class_<Trace>(m, "Trace")
      .def(py::init<>())
      .def_readwrite("events", &Trace::events)
      .def_readwrite("source_label", &Trace::source_label)
      .def_readwrite("reordered_on_load", &Trace::reordered_on_load);
  m.def("parse_trace", &parse_trace, py::arg("path"));
  m.def("parse_trace_text", &parse_trace_text, py::arg("text"), py::arg("label") = "<text>");
  m.def("serialize_trace", [](const Trace& t, const std::string& path) { serialize_trace(t, path); },
        py::arg("trace"), py::arg("path"));
  m.def("downscale", &downscale, py::arg("trace"), py::arg("factor"));
  m.def(
      "synth_burst",
      [](uint64_t seed, double base_rps, double burst_rps, int64_t burst_start_ms, int64_t burst_len_ms,
         int64_t total_ms, int prompt_tokens, int output_tokens) {
        return synth_burst(BurstSpec{seed, base_rps, burst_rps, burst_start_ms, burst_len_ms, total_ms,
                                     prompt_tokens, output_tokens});
      },
      py::arg("seed"), py::arg("base_rps"), py::arg("burst_rps"), py::arg("burst_start_ms"),
      py::arg("burst_len_ms"), py::arg("total_ms"), py::arg("prompt_tokens"), py::arg("output_tokens"));
  m.def("synth_gamma", &synth_gamma, py::arg("seed"), py::arg("rps"), py::arg("shape"), py::arg("total_ms"),
        py::arg("prompt_tokens"), py::arg("output_tokens"));
  m.def("synthetic_prompt", &synthetic_prompt, py::arg("seed"), py::arg("req"), py::arg("n"), py::arg("vocab"));

  py::class_<KvConfig>(m, "KvConfig")
      .def(py::init([](int bt, int64_t bb, int64_t cap) { return KvConfig{bt, bb, cap}; }),
           py::arg("block_tokens") = 16, py::arg("block_bytes") = 2 * 1024 * 1024,
           py::arg("static_capacity_blocks") = 1)
      .def_readwrite("block_tokens", &KvConfig::block_tokens)
      .def_readwrite("block_bytes", &KvConfig::block_bytes)
      .def_readwrite("static_capacity_blocks", &KvConfig::static_capacity_blocks);
  py::class_<KvBlockPool>(m, "KvBlockPool")
      .def(py::init<const KvConfig&>())
      .def("admit", &KvBlockPool::admit)
      .def("is_admitted", &KvBlockPool::is_admitted)
      .def("alloc_for_tokens", &KvBlockPool::alloc_for_tokens)
      .def("release", &KvBlockPool::release)
      .def("attach_blocks", &KvBlockPool::attach_blocks)
      .def("detach_blocks",
           [](KvBlockPool& p, int64_t n) {
             const DetachResult r = p.detach_blocks(n);
             return py::make_tuple(r.removed_now, r.deferred, r.capacity_blocks);
           })
      .def("preempt_victim",
           [](KvBlockPool& p, py::object eligible) {
             if (eligible.is_none()) return p.preempt_victim([](RequestId) { return true; });
             return p.preempt_victim([&](RequestId r) { return eligible(r).cast<bool>(); });
           },
           py::arg("eligible") = py::none())
      .def("capacity_blocks", &KvBlockPool::capacity_blocks)
      .def("free_blocks", &KvBlockPool::free_blocks)
      .def("used_blocks", &KvBlockPool::used_blocks)
      .def("attached_extra_blocks", &KvBlockPool::attached_extra_blocks)
      .def("pending_detach_blocks", &KvBlockPool::pending_detach_blocks)
      .def("tokens_of", &KvBlockPool::tokens_of)
      .def("blocks_of", &KvBlockPool::blocks_of)
      .def("block_list", &KvBlockPool::block_list)
      .def("usage_fraction", &KvBlockPool::usage_fraction)
      .def("take_retired", &KvBlockPool::take_retired)
      .def("check_invariants", &KvBlockPool::check_invariants);

  m.def("percentile_nearest_rank", &percentile_nearest_rank, py::arg("values"), py::arg("p"));
  m.def("decode_step_ms",
        [](const py::dict& engine, const std::vector<int>& bits, int64_t blocks) {
          std::vector<Precision> tags;
          for (int b : bits) tags.push_back(precision_from_bits(b));
          return engine_from(engine).cost.decode_step_ms(tags, blocks);
        });
  m.def("swap_duration_ms",
        [](const py::dict& engine, int64_t bytes) { return engine_from(engine).cost.swap_duration_ms(bytes); });
  m.def("auto_static_capacity_blocks",
        [](const py::dict& engine) { return engine_from(engine).auto_static_capacity_blocks(); });
  m.def("controller_defaults",
        [](const std::string& mode, int num_layers) {
          const ControllerConfig c = ControllerConfig::defaults_for(
              mode == "accuracy" ? ControllerMode::kAccuracy : ControllerMode::kPerformance, num_layers);
          py::dict d;
          d["enabled"] = c.enabled;
          d["mode"] = mode;
          d["kv_trigger"] = c.kv_trigger;
          d["kv_low"] = c.kv_low;
          d["queue_trigger_ms"] = c.queue_trigger_ms;
          d["hold_ms"] = c.hold_ms;
          d["max_swapped_layers"] = c.max_swapped_layers;
          d["swap_step"] = c.swap_step;
          d["telemetry_window_ms"] = c.telemetry_window_ms;
          d["target_bits"] = c.target_bits;
          return d;
        });
  m.def("validate_controller", [](const py::dict& d, int num_layers) { controller_from(d).validate(num_layers); });

  // engine: device = ms_ctx* as an integer (0 = no device, cost model only)
  m.def(
      "run_simulation",
      [](const py::dict& engine, const py::dict& arm, const Trace& trace, uint64_t seed, uintptr_t device,
         int vocab, const std::string& clock, bool record) {
        const ClockMode cm = clock == "device" ? ClockMode::kDevice : clock == "wall" ? ClockMode::kWall : ClockMode::kVirtual;
        if (clock != "device" && clock != "virtual" && clock != "wall")
          throw std::invalid_argument("clock must be virtual, device or wall");
        if (cm == ClockMode::kWall && device == 0) throw std::invalid_argument("wall clock needs a device");
        const EngineConfig ec = engine_from(engine);
        const ArmSpec as = arm_from(arm);
        if (device == 0) return result_dict(run_simulation(ec, as, trace, seed, nullptr, cm));
        CAbiBackend backend(reinterpret_cast<ms_ctx*>(device), vocab, cm != ClockMode::kVirtual);
        backend.set_recording(record, ec.model.num_layers);
        RunResult r;
        {
          py::gil_scoped_release nogil;
          r = run_simulation(ec, as, trace, seed, &backend, cm);
        }
        py::dict out = result_dict(r);
        if (record) {
          py::list calls;
          for (const auto& c : backend.calls()) {
            py::dict d;
            d["kind"] = std::string(1, c.kind);
            d["reqs"] = c.reqs;
            d["pos"] = c.pos;
            d["bits"] = c.bits;
            calls.append(d);
          }
          out["device_calls"] = calls;
        }
        return out;
      },
      py::arg("engine"), py::arg("arm"), py::arg("trace"), py::arg("seed"), py::arg("device") = 0,
      py::arg("vocab") = 0, py::arg("clock") = "virtual", py::arg("record") = false);
}
