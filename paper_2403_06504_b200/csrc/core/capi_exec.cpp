// B200 execution entry points of the C ABI:
//   offsim_execute      (include/offsim/offsim_c.h) scenario -> real run
//   fy_graph_execute    (include/fuyou/fy_adam.h)   same, with caller-owned
//                                                   per-chunk state buffers
// plus the JSON codecs of ExecOptions and ExecReport. A {"dry_run": true}
// option plans, maps and simulates without touching a GPU (CPU tests).

#include "capi_internal.hpp"

#include "fuyou/fy_adam.h"
#include "offsim/exec.hpp"
#include "offsim/runner.hpp"

#include <json.hpp>

#include <set>

namespace offsim {

using json = nlohmann::ordered_json;

namespace {

struct ParsedOptions {
    ExecOptions exec;
    bool dry_run = false;
    std::string variant;             // optional override
    std::string placement = "auto";  // checkpoint placement: auto | cpu | ssd
};

ParsedOptions parse_options(const char* text) {
    ParsedOptions out;
    if (!text || !*text) return out;
    json doc;
    try {
        doc = json::parse(text);
    } catch (const json::parse_error& e) {
        throw ConfigError(std::string("exec options parse error: ") + e.what());
    }
    if (!doc.is_object()) throw ConfigError("exec options must be an object");
    static const std::set<std::string> keys = {"device", "tier", "file_dir", "direct_io",
                                               "compute_rate", "state_slots", "seed",
                                               "verify_swaps", "adam", "dry_run", "variant",
                                               "swap_only", "max_blocks", "placement",
                                               "compute_mode", "host_ring", "checksum_states",
                                               "resident_groups", "fixed_buffers", "io_depth",
                                               "launch", "warm_files"};
    for (const auto& it : doc.items())
        if (!keys.count(it.key())) throw ConfigError("unknown key '" + it.key() + "' in exec options");
    try {
        ExecOptions& o = out.exec;
        o.device = doc.value("device", o.device);
        const std::string tier = doc.value("tier", std::string("host"));
        if (tier == "host") o.tier = StateTier::host;
        else if (tier == "file") o.tier = StateTier::file;
        else throw ConfigError("exec options: tier must be 'host' or 'file'");
        if (doc.contains("file_dir") && doc["file_dir"].is_array()) {
            // one directory per SSD: the tier files are striped over them
            for (const auto& d : doc["file_dir"]) o.file_dirs.push_back(d.get<std::string>());
            if (o.file_dirs.empty()) throw ConfigError("exec options: file_dir list is empty");
            if (o.file_dirs.size() > 64) throw ConfigError("exec options: at most 64 file_dir entries");
            if (std::set<std::string>(o.file_dirs.begin(), o.file_dirs.end()).size() != o.file_dirs.size())
                throw ConfigError("exec options: file_dir entries must be distinct");
            o.file_dir = o.file_dirs.front();
        } else {
            o.file_dir = doc.value("file_dir", o.file_dir);
        }
        o.direct_io = doc.value("direct_io", o.direct_io);
        o.fixed_buffers = doc.value("fixed_buffers", o.fixed_buffers);
        o.io_depth = doc.value("io_depth", o.io_depth);
        o.warm_files = doc.value("warm_files", o.warm_files);
        o.launch = doc.value("launch", o.launch);
        if (o.launch != "graph" && o.launch != "stream")
            throw ConfigError("exec options: launch must be \"graph\" or \"stream\"");
        if (o.io_depth < 1 || o.io_depth > 1024) throw ConfigError("exec options: io_depth must be 1..1024");
        o.compute_rate = doc.value("compute_rate", o.compute_rate);
        o.state_slots = doc.value("state_slots", o.state_slots);
        o.seed = doc.value("seed", o.seed);
        o.verify_swaps = doc.value("verify_swaps", o.verify_swaps);
        out.dry_run = doc.value("dry_run", false);
        out.variant = doc.value("variant", std::string());
        o.compute_mode = doc.value("compute_mode", o.compute_mode);
        if (doc.contains("host_ring") && doc.at("host_ring").is_string()) {
            if (doc.at("host_ring").get<std::string>() != "auto")
                throw ConfigError("exec options: host_ring must be a slot count or 'auto'");
            o.host_ring_auto = true;
        } else {
            o.host_ring = doc.value("host_ring", o.host_ring);
        }
        o.checksum_states = doc.value("checksum_states", o.checksum_states);
        if (doc.contains("resident_groups") && doc.at("resident_groups").is_string()) {
            const std::string v = doc.at("resident_groups").get<std::string>();
            if (v != "all" && v != "auto")
                throw ConfigError("exec options: resident_groups must be a count, 'all' or 'auto'");
            o.resident_groups = v == "all" ? 0xffffffffu : kResidentAuto;
        } else {
            o.resident_groups = doc.value("resident_groups", o.resident_groups);
        }
        o.swap_only = doc.value("swap_only", o.swap_only);
        o.max_blocks = doc.value("max_blocks", o.max_blocks);
        out.placement = doc.value("placement", out.placement);
        if (out.placement != "auto" && out.placement != "cpu" && out.placement != "ssd")
            throw ConfigError("exec options: placement must be 'auto', 'cpu' or 'ssd'");
        if (doc.contains("adam")) {
            const json& a = doc.at("adam");
            static const std::set<std::string> akeys = {"lr", "beta1", "beta2", "eps", "weight_decay",
                                                        "step", "adamw_mode", "bias_correction",
                                                        "grad_scale"};
            for (const auto& it : a.items())
                if (!akeys.count(it.key())) throw ConfigError("unknown key '" + it.key() + "' in exec options.adam");
            AdamHyper& h = o.adam;
            h.lr = a.value("lr", h.lr);
            h.beta1 = a.value("beta1", h.beta1);
            h.beta2 = a.value("beta2", h.beta2);
            h.eps = a.value("eps", h.eps);
            h.weight_decay = a.value("weight_decay", h.weight_decay);
            h.step = a.value("step", h.step);
            h.adamw_mode = a.value("adamw_mode", h.adamw_mode);
            h.bias_correction = a.value("bias_correction", h.bias_correction);
            h.grad_scale = a.value("grad_scale", h.grad_scale);
            if (h.step < 1) throw ConfigError("exec options: adam.step must be >= 1");
        }
        if (o.state_slots < 2) throw ConfigError("exec options: state_slots must be >= 2");
    } catch (const json::exception& e) {
        throw ConfigError(std::string("exec options: bad value: ") + e.what());
    }
    return out;
}

json bytes_json(const std::map<std::string, double>& m) {
    json j = json::object();
    for (const auto& [k, v] : m) j[k] = v;
    return j;
}

json rings_json(const RingDepths& d) {
    return json{{"states", d.states}, {"params", d.params}, {"weights", d.weights}, {"acts", d.acts}};
}

json trace_stats(const SimTrace& t) {
    json busy = json::object();
    for (const auto& [lane, ns] : t.busy_ns) busy[to_string(lane)] = static_cast<double>(ns) * 1e-9;
    json peaks = json::object();
    for (const auto& [pool, b] : t.peak_mem) peaks[to_string(pool)] = b;
    return json{{"makespan_s", t.makespan_s()}, {"busy_s", busy}, {"peak_mem_bytes", peaks}};
}

// Per optimizer group: real timings of its hops (state_h2d -> update ->
// state_d2h/param_d2h), the evidence for overlap with backward.
json optimizer_json(const ExecReport& r) {
    double upd_ns = 0, n_upd = 0, params = 0;
    std::uint64_t first = ~0ull, last = 0;
    std::map<std::uint32_t, const TraceEvent*> ev;
    for (const TraceEvent& e : r.trace.events) ev[e.task_id] = &e;
    for (const Task& t : r.graph.tasks) {
        if (t.kind != TaskKind::optimizer_update) continue;
        const TraceEvent* e = ev.at(t.id);
        upd_ns += static_cast<double>(e->end_ns - e->start_ns);
        n_upd += 1;
        params += t.work;
        first = std::min(first, e->start_ns);
        last = std::max(last, e->end_ns);
    }
    return json{{"groups", n_upd},
                {"params", params},
                {"kernel_time_s", upd_ns * 1e-9},
                {"kernel_params_per_s", upd_ns > 0 ? params / (upd_ns * 1e-9) : 0.0},
                {"window_s", last > first ? static_cast<double>(last - first) * 1e-9 : 0.0},
                {"grad_sq_sum", r.grad_sq_sum},
                {"expected_grad_sq_sum", r.expected_grad_sq_sum},
                {"nonfinite", r.nonfinite}};
}

// Executed time and bytes per (lane, direction, payload) leg, from the real
// trace: the SSD lane's reads and writes are timed as separate legs (each
// event is one request's own duration), not split by bytes.
json legs_json(const ExecReport& r) {
    struct Leg {
        double bytes = 0, busy_ns = 0, count = 0;
    };
    std::map<std::string, Leg> legs;
    for (const TraceEvent& e : r.trace.events) {
        if (e.dir == TransferDir::none || e.work <= 0.0) continue;
        Leg& l = legs[std::string(to_string(e.resource)) + "/" + to_string(e.dir) + "/" + to_string(e.payload)];
        l.bytes += e.work;
        l.busy_ns += static_cast<double>(e.end_ns - e.start_ns);
        l.count += 1;
    }
    json j = json::object();
    for (const auto& [k, l] : legs)
        j[k] = json{{"bytes", l.bytes}, {"busy_s", l.busy_ns * 1e-9}, {"requests", l.count},
                    {"gbs", l.busy_ns > 0 ? l.bytes / l.busy_ns : 0.0}};
    return j;
}

json rates_json(const MeasuredRates& m) {
    return json{{"h2d_bps", m.h2d_bps},
                {"d2h_bps", m.d2h_bps},
                {"h2d_effective_bps", m.h2d_effective_bps},
                {"d2h_effective_bps", m.d2h_effective_bps},
                {"h2d_simplex_effective_bps", m.h2d_simplex_effective_bps},
                {"d2h_simplex_effective_bps", m.d2h_simplex_effective_bps},
                {"c2g_overlap", m.c2g_overlap},
                {"g2c_overlap", m.g2c_overlap},
                {"file_read_bps", m.file_read_bps},
                {"file_write_bps", m.file_write_bps},
                {"file_read_effective_bps", m.file_read_effective_bps},
                {"file_write_effective_bps", m.file_write_effective_bps},
                {"file_read_loaded_bps", m.file_read_loaded_bps},
                {"file_write_loaded_bps", m.file_write_loaded_bps},
                {"ssd_link_overlap", m.ssd_link_overlap},
                {"optimizer_params_per_s", m.optimizer_params_per_s},
                {"compute_flops", m.compute_flops / m.compute_headroom},
                {"compute_effective_flops", m.compute_effective_flops}};
}

json analytic_json(const TaskGraph& g, const HardwareConfig& hw, double executed_s) {
    const AnalyticTimes a = analytic_iteration(g, hw);
    return json{{"t_f_s", a.t_f},
                {"t_bo_s", a.t_bo},
                {"t_iter_s", a.t_iter},
                {"bottleneck_f", a.bottleneck_f},
                {"bottleneck_bo", a.bottleneck_bo},
                {"executed_over_analytic", a.t_iter > 0 ? executed_s / a.t_iter : 0.0}};
}

} // namespace

std::string exec_summary_json(const ExecReport& r) {
    json checks = json::array();
    for (const auto& e : r.invariants.entries)
        checks.push_back(json{{"name", e.name}, {"pass", e.pass}, {"detail", e.detail}});
    const HardwareConfig& h = r.hw_exec;
    const HardwareConfig& e = r.hw_predicted;
    const double pred_s = static_cast<double>(r.predicted.makespan_ns) * 1e-9;
    const double exec_s = r.trace.makespan_s();
    const json doc = {
        {"schema_version", 1},
        {"command", "execute"},
        {"variant", to_string(r.graph.header.variant)},
        {"checkpoint_location", r.graph.header.checkpoint_location},
        {"task_count", r.graph.tasks.size()},
        {"hw_exec", json{{"bw_gpu", h.bw_gpu}, {"bw_s2c", h.bw_s2c}, {"bw_c2s", h.bw_c2s},
                         {"cpu_opt_tput", h.cpu_opt_tput}, {"gpu_tput", h.gpu_tput},
                         {"gpu_mem", h.gpu_mem}, {"cpu_mem", h.cpu_mem}}},
        {"executed", trace_stats(r.trace)},
        {"planned", trace_stats(r.planned)},
        {"hw_predicted", json{{"bw_gpu", e.bw_gpu}, {"bw_s2c", e.bw_s2c}, {"bw_c2s", e.bw_c2s},
                              {"cpu_opt_tput", e.cpu_opt_tput}, {"gpu_tput", e.gpu_tput}}},
        {"predicted", trace_stats(r.predicted)},
        {"executed_over_predicted",
         pred_s > 0 ? static_cast<double>(r.trace.makespan_ns) * 1e-9 / pred_s : 0.0},
        {"measured_rates", rates_json(r.rates)},
        // the calibration loop: analytic t_iter (reference cost-model
        // structure) and the DES, on the in-run effective rates and on the
        // scenario's own hardware (a persisted measured preset, or the
        // modeled preset the plan was made on)
        {"analytic", analytic_json(r.graph, e, exec_s)},
        {"scenario_prediction",
         json{{"hardware", r.hw_scenario.name},
              {"des_makespan_s", r.scenario_predicted.makespan_s()},
              {"executed_over_des", r.scenario_predicted.makespan_ns > 0
                                        ? exec_s / r.scenario_predicted.makespan_s() : 0.0},
              {"analytic", analytic_json(r.graph, r.hw_scenario, exec_s)}}},
        // the invariant check's roofline uses hw_exec = measured burst rates
        // x headroom (b200_hardware); the same bound on the effective rates,
        // with no headroom, is reported beside it
        {"roofline_check",
         json{{"headroom", json{{"link", 1.05}, {"file", 1.5}, {"optimizer", 1.05}}},
              {"bound_exec_s", static_cast<double>(roofline_lower_bound_ns(r.graph, r.hw_exec)) * 1e-9},
              {"bound_effective_s", static_cast<double>(roofline_lower_bound_ns(r.graph, e)) * 1e-9},
              {"executed_s", exec_s}}},
        {"legs", legs_json(r)},
        {"optimizer", optimizer_json(r)},
        {"reference_bytes", bytes_json(r.reference_bytes)},
        {"physical_bytes", bytes_json(r.physical_bytes)},
        {"swap_checks", r.swap_checks},
        {"swap_mismatches", r.swap_mismatches},
        {"kernel_launches", r.kernel_launches},
        {"io_engine", r.io_engine},
        {"file_devices", r.file_devices},
        {"io_requests", {{"registered_bytes", r.io_registered_bytes},
                         {"fixed", r.io_fixed_requests},
                         {"plain", r.io_plain_requests}}},
        {"file_warmup_s", r.file_warmup_s},
        {"pinned_host_bytes", r.pinned_host_bytes},
        {"host_ring", rings_json(r.host_ring)},
        {"state_checksum", r.state_checksum},
        {"resident_groups", r.resident_groups},
        {"launch", r.launch_mode},
        {"invariants", checks},
        {"all_invariants_pass", r.invariants.all_pass && r.swap_mismatches == 0},
    };
    return doc.dump(2) + "\n";
}

namespace {

// The unchanged planner; `placement` only overrides the all-or-nothing
// checkpoint placement input (runner.cpp:90-106), e.g. to force the
// GPU->host->SSD leg of the swap path.
SwapPlan plan_with_placement(const Scenario& s, const std::string& placement) {
    if (placement == "auto") return plan_for_scenario(s);
    PlannerOptions o;
    o.mode = s.planner_mode;
    o.fixed_d_f_bytes = s.planner_value;
    o.fixed_coefficient = s.planner_value;
    o.checkpoints_on_ssd = placement == "ssd";
    return plan_swaps(s.model, s.hardware, o);
}

// Dry run: the mapped graph and its DES on nominal B200 rates (no GPU);
// trace_out (optional) receives that DES trace as a Chrome trace.
std::string dry_run_json(const Scenario& s, const ParsedOptions& po, ScheduleVariant v,
                         std::string* trace_out = nullptr) {
    const SwapPlan plan = plan_with_placement(s, po.placement);
    const TaskGraph ref = build_schedule(s.model, s.hardware, plan, v);
    TaskGraph mapped = map_graph_for_b200(ref, po.exec.tier, po.exec.state_slots,
                                          po.exec.resident_groups == kResidentAuto ? 0 : po.exec.resident_groups);
    if (po.exec.swap_only) mapped = swap_subgraph(mapped, po.exec.max_blocks);
    const RingDepths rings = host_ring_depths(mapped, po.exec);
    add_host_ring_edges(mapped, rings);
    MeasuredRates nominal;
    nominal.h2d_bps = nominal.d2h_bps = 55e9;
    nominal.file_read_bps = nominal.file_write_bps = po.exec.tier == StateTier::file ? 2e9 : 0.0;
    nominal.optimizer_params_per_s = 2.1e11;
    nominal.compute_flops = po.exec.compute_rate > 0 ? po.exec.compute_rate : s.hardware.gpu_tput;
    nominal.gpu_mem = 180ull * 1000 * 1000 * 1000;
    nominal.cpu_mem = 2000ull * 1000 * 1000 * 1000;
    const HardwareConfig hw = b200_hardware(s.hardware, nominal);
    const SimTrace tr = simulate(mapped, hw);
    const InvariantReport inv = check_trace_invariants(mapped, tr, hw);
    if (trace_out) *trace_out = to_chrome_trace_json(mapped, tr);
    MeasuredRates overlap;
    link_overlap(mapped, tr, overlap);
    std::map<std::string, double> ref_bytes, mapped_bytes;
    for (const Task& t : ref.tasks)
        if (t.kind == TaskKind::transfer)
            ref_bytes[std::string(to_string(t.resource)) + "/" + to_string(t.payload)] += t.work;
    json inserted = json::array();
    for (const Task& t : mapped.tasks) {
        if (t.kind == TaskKind::transfer)
            mapped_bytes[std::string(to_string(t.resource)) + "/" + to_string(t.payload)] += t.work;
        if (t.name.find("_h2d ") != std::string::npos || t.name.find("_d2h ") != std::string::npos)
            inserted.push_back(t.name);
    }
    json checks = json::array();
    for (const auto& e : inv.entries)
        checks.push_back(json{{"name", e.name}, {"pass", e.pass}, {"detail", e.detail}});
    const json doc = {{"schema_version", 1},
                      {"command", "execute"},
                      {"dry_run", true},
                      {"variant", to_string(v)},
                      {"reference_task_count", ref.tasks.size()},
                      {"task_count", mapped.tasks.size()},
                      {"inserted_tasks", inserted},
                      {"host_ring", rings_json(rings)},
                      {"windows", json{{"prefetch_window_layers", mapped.header.prefetch_window_layers},
                                       {"offload_window_blocks", mapped.header.offload_window_blocks},
                                       {"cpu_stage_window_layers", mapped.header.cpu_stage_window_layers}}},
                      {"reference_bytes", bytes_json(ref_bytes)},
                      {"mapped_bytes", bytes_json(mapped_bytes)},
                      {"planned", trace_stats(tr)},
                      {"analytic", analytic_json(mapped, hw, tr.makespan_s())},
                      {"link_overlap", json{{"c2g", overlap.c2g_overlap},
                                            {"g2c", overlap.g2c_overlap},
                                            {"ssd_link", overlap.ssd_link_overlap},
                                            {"c2g_bytes", overlap.c2g_bytes},
                                            {"g2c_bytes", overlap.g2c_bytes}}},
                      {"invariants", checks},
                      {"all_invariants_pass", inv.all_pass}};
    return doc.dump(2) + "\n";
}

offsim_status run_exec(const Scenario& s, const char* opts_json,
                       const std::vector<ChunkBuffers>* chunks, char** summary_out,
                       char** trace_out) {
    const ParsedOptions po = parse_options(opts_json);
    const ScheduleVariant v =
        po.variant.empty() ? s.variant : schedule_variant_from_string(po.variant);
    Scenario sv = s;
    sv.variant = v;
    if (po.dry_run) {
        std::string trace;
        *summary_out = capi::copy_out(dry_run_json(sv, po, v, trace_out ? &trace : nullptr));
        if (trace_out) *trace_out = capi::copy_out(trace);
        return OFFSIM_OK;
    }
    const SwapPlan plan = plan_with_placement(sv, po.placement);
    const ExecReport rep = execute(sv.model, sv.hardware, plan, v, po.exec, chunks);
    const std::string summary = exec_summary_json(rep);
    *summary_out = capi::copy_out(summary);
    if (trace_out) *trace_out = capi::copy_out(to_chrome_trace_json(rep.graph, rep.trace));
    if (!rep.invariants.all_pass || rep.swap_mismatches != 0)
        return capi::fail(OFFSIM_ERR_INVARIANT, "executed trace failed its checks; see summary");
    return OFFSIM_OK;
}

} // namespace

} // namespace offsim

extern "C" {

offsim_status offsim_execute(const offsim_scenario* s, const char* exec_opts_json,
                             char** summary_json_out, char** trace_json_out) {
    if (!s || !summary_json_out) return offsim::capi::fail(OFFSIM_ERR_CONFIG, "null argument");
    return offsim::capi::guarded([&] {
        return offsim::run_exec(s->scenario, exec_opts_json, nullptr, summary_json_out, trace_json_out);
    });
}

fy_status fy_graph_execute(const char* scenario_json, const char* exec_opts_json,
                           const fy_chunk* chunks, uint32_t chunk_count, char** summary_json_out) {
    if (!scenario_json || !summary_json_out || (chunk_count && !chunks))
        return static_cast<fy_status>(offsim::capi::fail(OFFSIM_ERR_CONFIG, "null argument"));
    const offsim_status st = offsim::capi::guarded([&] {
        const offsim::Scenario sc = offsim::load_scenario(scenario_json);
        std::vector<offsim::ChunkBuffers> bufs;
        for (uint32_t k = 0; k < chunk_count; ++k) {
            if (chunks[k].n != 12ull * sc.model.hidden_dim * sc.model.hidden_dim)
                throw offsim::ConfigError("fy_graph_execute: chunk " + std::to_string(k) +
                                          " size differs from 12*h^2");
            if (chunks[k].flags != 0)
                throw offsim::ConfigError("fy_graph_execute: chunk " + std::to_string(k) +
                                          ": chunk flags are a pipeline feature");
            if (chunks[k].states_stride != 0 && chunks[k].states_stride != chunks[k].n)
                throw offsim::ConfigError("fy_graph_execute: chunk " + std::to_string(k) +
                                          ": strided states are a pipeline feature (contiguous here)");
            bufs.push_back({chunks[k].h_states, chunks[k].h_param, chunks[k].grad});
        }
        return offsim::run_exec(sc, exec_opts_json, chunk_count ? &bufs : nullptr, summary_json_out,
                                nullptr);
    });
    return static_cast<fy_status>(st);
}

} // extern "C"
