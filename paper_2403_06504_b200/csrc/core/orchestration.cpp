// Scenario documents, capacity analysis and the runner — restates
// proj/src/scenario.cpp, proj/src/capacity.cpp and proj/src/runner.cpp.
// Report layouts (key order, number formatting via nlohmann::ordered_json,
// %.9g in CSVs) are kept identical so the C ABI returns byte-identical
// documents (tests/parity).

#include "offsim/capacity.hpp"
#include "offsim/errors.hpp"
#include "offsim/presets.hpp"
#include "offsim/runner.hpp"
#include "offsim/scenario.hpp"

#include <json.hpp>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <set>
#include <sstream>
#include <thread>

namespace offsim {

using json = nlohmann::ordered_json;

// ================================================================ scenario

namespace {

void only_keys(const json& obj, const std::set<std::string>& allowed, const std::string& where) {
    for (const auto& item : obj.items())
        if (!allowed.count(item.key()))
            throw ConfigError("unknown key '" + item.key() + "' in " + where);
}

template <typename T>
void take(const json& obj, const char* key, T& dst) {
    const auto it = obj.find(key);
    if (it == obj.end()) return;
    try {
        dst = it->template get<T>();
    } catch (const json::exception&) {
        throw ConfigError(std::string("bad value for key '") + key + "'");
    }
}

void require_keys(const json& obj, std::initializer_list<const char*> keys, const char* where) {
    for (const char* k : keys)
        if (!obj.contains(k)) throw ConfigError(std::string(where) + ": missing key '" + k + "'");
}

ModelConfig model_from(const json& node) {
    if (node.is_string()) return model_preset(node.get<std::string>());
    if (!node.is_object()) throw ConfigError("'model' must be a preset name or an object");
    only_keys(node,
              {"preset", "name", "num_layers", "num_heads", "hidden_dim", "batch_size", "seq_len",
               "param_elem_bytes", "optimizer_state_multiplier", "activation_elem_bytes",
               "extra_flops_per_block"},
              "model");
    ModelConfig m;
    if (node.contains("preset"))
        m = model_preset(node.at("preset").get<std::string>());
    else
        require_keys(node, {"num_layers", "num_heads", "hidden_dim"}, "model");
    take(node, "name", m.name);
    take(node, "num_layers", m.num_layers);
    take(node, "num_heads", m.num_heads);
    take(node, "hidden_dim", m.hidden_dim);
    take(node, "batch_size", m.batch_size);
    take(node, "seq_len", m.seq_len);
    take(node, "param_elem_bytes", m.param_elem_bytes);
    take(node, "optimizer_state_multiplier", m.optimizer_state_multiplier);
    take(node, "activation_elem_bytes", m.activation_elem_bytes);
    take(node, "extra_flops_per_block", m.extra_flops_per_block);
    m.validate();
    return m;
}

HardwareConfig hardware_from(const json& node) {
    if (node.is_string()) return hardware_preset(node.get<std::string>());
    if (!node.is_object()) throw ConfigError("'hardware' must be a preset name or an object");
    only_keys(node,
              {"preset", "name", "bw_gpu", "bw_s2c", "bw_c2s", "n_ssd", "gpu_mem", "cpu_mem",
               "ssd_capacity", "gpu_tput", "cpu_opt_tput", "gpu_price_dollars",
               "ssd_price_dollars", "server_price_dollars"},
              "hardware");
    HardwareConfig hw;
    if (node.contains("preset"))
        hw = hardware_preset(node.at("preset").get<std::string>());
    else
        require_keys(node,
                     {"bw_gpu", "bw_s2c", "bw_c2s", "gpu_mem", "cpu_mem", "ssd_capacity",
                      "gpu_tput", "cpu_opt_tput"},
                     "hardware");
    take(node, "name", hw.name);
    take(node, "bw_gpu", hw.bw_gpu);
    take(node, "bw_s2c", hw.bw_s2c);
    take(node, "bw_c2s", hw.bw_c2s);
    take(node, "n_ssd", hw.n_ssd);
    take(node, "gpu_mem", hw.gpu_mem);
    take(node, "cpu_mem", hw.cpu_mem);
    take(node, "ssd_capacity", hw.ssd_capacity);
    take(node, "gpu_tput", hw.gpu_tput);
    take(node, "cpu_opt_tput", hw.cpu_opt_tput);
    take(node, "gpu_price_dollars", hw.gpu_price_dollars);
    take(node, "ssd_price_dollars", hw.ssd_price_dollars);
    take(node, "server_price_dollars", hw.server_price_dollars);
    if (const ValidationReport r = validate(hw); !r.ok())
        throw ConfigError("hardware: " + r.errors.front());
    return hw;
}

void planner_from(const json& node, Scenario& s) {
    if (!node.is_object()) throw ConfigError("'planner' must be an object");
    only_keys(node, {"mode", "d_f", "coefficient"}, "planner");
    const std::string mode = node.value("mode", std::string("auto"));
    if (mode == "auto") {
        s.planner_mode = PlannerOptions::Mode::automatic;
        if (node.contains("d_f") || node.contains("coefficient"))
            throw ConfigError("planner: mode 'auto' takes no value");
        return;
    }
    if (mode == "fixed_d_f") {
        s.planner_mode = PlannerOptions::Mode::fixed_d_f;
        if (!node.contains("d_f")) throw ConfigError("planner: mode 'fixed_d_f' needs 'd_f'");
        s.planner_value = node.at("d_f").get<double>();
        return;
    }
    if (mode == "fixed_coefficient") {
        s.planner_mode = PlannerOptions::Mode::fixed_coefficient;
        if (!node.contains("coefficient"))
            throw ConfigError("planner: mode 'fixed_coefficient' needs 'coefficient'");
        s.planner_value = node.at("coefficient").get<double>();
        if (s.planner_value < 0.0 || s.planner_value > 1.0)
            throw ConfigError("planner: coefficient must be in [0, 1]");
        return;
    }
    throw ConfigError("planner: unknown mode '" + mode + "'");
}

struct PresetRow {
    const char* name;
    const char* model;
    const char* machine;
    std::uint64_t batch;
};
constexpr PresetRow kPresetRows[] = {
    {"13b-a100-b8", "gpt3-13b", "a100-12ssd", 8},
    {"13b-a100-b16", "gpt3-13b", "a100-12ssd", 16},
    {"13b-a100-b32", "gpt3-13b", "a100-12ssd", 32},
    {"13b-a100-b64", "gpt3-13b", "a100-12ssd", 64},
    {"13b-a100-b80", "gpt3-13b", "a100-12ssd", 80},
    {"13b-4090-b32", "gpt3-13b", "rtx4090-12ssd", 32},
    {"175b-a100-b16", "gpt3-175b", "a100-12ssd", 16},
    {"175b-4090-b8", "gpt3-175b", "rtx4090-12ssd", 8},
};

} // namespace

Scenario load_scenario(const std::string& json_text) {
    json doc;
    try {
        doc = json::parse(json_text);
    } catch (const json::parse_error& e) {
        throw ConfigError(std::string("scenario parse error: ") + e.what());
    }
    if (!doc.is_object()) throw ConfigError("scenario document must be an object");
    only_keys(doc, {"schema_version", "model", "hardware", "variant", "planner", "seed"},
              "scenario");
    Scenario s;
    if (!doc.contains("schema_version")) throw ConfigError("scenario: missing key 'schema_version'");
    s.schema_version = doc.at("schema_version").get<int>();
    if (s.schema_version != kScenarioSchemaVersion)
        throw ConfigError("scenario: unsupported schema_version " + std::to_string(s.schema_version));
    require_keys(doc, {"model", "hardware"}, "scenario");
    s.model = model_from(doc.at("model"));
    s.hardware = hardware_from(doc.at("hardware"));
    if (doc.contains("variant"))
        s.variant = schedule_variant_from_string(doc.at("variant").get<std::string>());
    if (doc.contains("planner")) planner_from(doc.at("planner"), s);
    if (doc.contains("seed")) s.seed = doc.at("seed").get<std::int64_t>();
    return s;
}

std::string scenario_to_json(const Scenario& s) {
    const ModelConfig& m = s.model;
    const HardwareConfig& h = s.hardware;
    json planner;
    if (s.planner_mode == PlannerOptions::Mode::fixed_d_f)
        planner = {{"mode", "fixed_d_f"}, {"d_f", s.planner_value}};
    else if (s.planner_mode == PlannerOptions::Mode::fixed_coefficient)
        planner = {{"mode", "fixed_coefficient"}, {"coefficient", s.planner_value}};
    else
        planner = {{"mode", "auto"}};
    const json doc = {
        {"schema_version", s.schema_version},
        {"model",
         {{"name", m.name},
          {"num_layers", m.num_layers},
          {"num_heads", m.num_heads},
          {"hidden_dim", m.hidden_dim},
          {"batch_size", m.batch_size},
          {"seq_len", m.seq_len},
          {"param_elem_bytes", m.param_elem_bytes},
          {"optimizer_state_multiplier", m.optimizer_state_multiplier},
          {"activation_elem_bytes", m.activation_elem_bytes},
          {"extra_flops_per_block", m.extra_flops_per_block}}},
        {"hardware",
         {{"name", h.name},
          {"bw_gpu", h.bw_gpu},
          {"bw_s2c", h.bw_s2c},
          {"bw_c2s", h.bw_c2s},
          {"n_ssd", h.n_ssd},
          {"gpu_mem", h.gpu_mem},
          {"cpu_mem", h.cpu_mem},
          {"ssd_capacity", h.ssd_capacity},
          {"gpu_tput", h.gpu_tput},
          {"cpu_opt_tput", h.cpu_opt_tput},
          {"gpu_price_dollars", h.gpu_price_dollars},
          {"ssd_price_dollars", h.ssd_price_dollars},
          {"server_price_dollars", h.server_price_dollars}}},
        {"variant", to_string(s.variant)},
        {"planner", planner},
        {"seed", s.seed},
    };
    return doc.dump(2) + "\n";
}

const std::vector<std::string>& scenario_preset_names() {
    static const std::vector<std::string> names = [] {
        std::vector<std::string> v;
        for (const PresetRow& r : kPresetRows) v.emplace_back(r.name);
        return v;
    }();
    return names;
}

Scenario scenario_preset(const std::string& name) {
    for (const PresetRow& r : kPresetRows) {
        if (name != r.name) continue;
        Scenario s;
        s.model = model_preset(r.model);
        s.model.batch_size = r.batch;
        s.hardware = hardware_preset(r.machine);
        return s;
    }
    throw ConfigError("unknown scenario preset '" + name + "'");
}

// ================================================================ capacity

const char* to_string(PolicyId id) {
    return id == PolicyId::zero_infinity ? "zero-infinity"
           : id == PolicyId::two_level   ? "two-level"
                                         : "unknown";
}

PolicyId policy_from_string(const std::string& s) {
    if (s == "zero-infinity") return PolicyId::zero_infinity;
    if (s == "two-level") return PolicyId::two_level;
    throw ConfigError("unknown placement policy '" + s + "'");
}

const char* to_string(CapacityBottleneck b) {
    switch (b) {
    case CapacityBottleneck::none: return "none";
    case CapacityBottleneck::ssd: return "ssd";
    case CapacityBottleneck::cpu_mem: return "cpu_mem";
    case CapacityBottleneck::gpu_mem: return "gpu_mem";
    }
    return "unknown";
}

namespace {

// Params + grads + optimizer states of kCpuStagingGroups streamed groups.
std::uint64_t staging_bytes(const ModelConfig& m) {
    const double block16 = 12.0 * static_cast<double>(m.hidden_dim) *
                           static_cast<double>(m.hidden_dim) *
                           static_cast<double>(m.param_elem_bytes);
    return static_cast<std::uint64_t>(
        std::llround(kCpuStagingGroups * block16 * (2.0 + m.optimizer_state_multiplier)));
}

} // namespace

PlacementBudget placement_budget(PolicyId policy, const ModelConfig& model,
                                 const HardwareConfig& hw) {
    const FootprintReport fp = footprint(model);
    PlacementBudget b;
    b.gpu_bytes = gpu_working_set_bytes(model);
    if (policy == PolicyId::zero_infinity) {
        b.ssd_bytes = fp.model_state_bytes;
        b.cpu_bytes = fp.total_checkpoint_bytes +
                      static_cast<std::uint64_t>(std::llround(
                          kZeroInfinityCpuBytesPerParam * static_cast<double>(fp.total_params)));
        b.checkpoints_on_ssd = false;
        return b;
    }
    const std::uint64_t stage = staging_bytes(model);
    const bool in_cpu = stage <= hw.cpu_mem && fp.total_checkpoint_bytes <= hw.cpu_mem - stage;
    b.checkpoints_on_ssd = !in_cpu;
    b.cpu_bytes = stage + (in_cpu ? fp.total_checkpoint_bytes : 0);
    b.ssd_bytes = fp.model_state_bytes + (in_cpu ? 0 : fp.total_checkpoint_bytes);
    return b;
}

Feasibility feasible(PolicyId policy, const ModelConfig& model, const HardwareConfig& hw) {
    const PlacementBudget b = placement_budget(policy, model, hw);
    const struct {
        CapacityBottleneck where;
        std::uint64_t need, have;
    } checks[] = {{CapacityBottleneck::ssd, b.ssd_bytes, hw.ssd_capacity},
                  {CapacityBottleneck::cpu_mem, b.cpu_bytes, hw.cpu_mem},
                  {CapacityBottleneck::gpu_mem, b.gpu_bytes, hw.gpu_mem}};
    Feasibility f;
    for (const auto& c : checks) {
        if (c.need <= c.have) continue;
        f.ok = false;
        f.bottleneck = c.where;
        std::ostringstream os;
        os << to_string(c.where) << ": needs " << c.need << " bytes, capacity " << c.have;
        f.detail = os.str();
        return f;
    }
    f.ok = true;
    f.bottleneck = CapacityBottleneck::none;
    return f;
}

MaxTrainable max_trainable(PolicyId policy, const HardwareConfig& hw,
                           const std::vector<ModelConfig>& candidates) {
    MaxTrainable out;
    CapacityBottleneck blocker = CapacityBottleneck::none;
    for (auto it = candidates.rbegin(); it != candidates.rend(); ++it) {
        const Feasibility f = feasible(policy, *it, hw);
        if (f.ok) {
            out.found = true;
            out.model = *it;
            out.limit = blocker;
            return out;
        }
        blocker = f.bottleneck;
    }
    out.limit = blocker;
    return out;
}

PriceTable price_table(const HardwareConfig& hw) {
    return PriceTable{hw.gpu_price_dollars, hw.ssd_price_dollars, hw.server_price_dollars};
}

double tokens_per_second(const ModelConfig& model, double t_iter_s) {
    if (t_iter_s <= 0.0) throw ConfigError("tokens_per_second: iteration time must be > 0");
    return static_cast<double>(model.batch_size) * static_cast<double>(model.seq_len) / t_iter_s;
}

double cost_effectiveness(double t_iter_s, const ModelConfig& model, const PriceTable& prices,
                          PriceScope scope, std::uint32_t n_ssd) {
    if (prices.gpu <= 0.0) throw ConfigError("cost_effectiveness: gpu price must be > 0");
    if (prices.ssd <= 0.0) throw ConfigError("cost_effectiveness: ssd price must be > 0");
    double dollars = prices.gpu + prices.ssd * static_cast<double>(n_ssd);
    if (scope == PriceScope::whole_server) {
        if (prices.server <= 0.0) throw ConfigError("cost_effectiveness: server price must be > 0");
        dollars += prices.server;
    }
    return tokens_per_second(model, t_iter_s) / dollars;
}

// ================================================================== runner

namespace {

std::string g9(double v) {
    char buf[48];
    std::snprintf(buf, sizeof buf, "%.9g", v);
    return buf;
}

json breakdown_json(const CostBreakdown& c) {
    return json{{"t_f_comp_s", c.t_f_comp},       {"t_f_gpu_s", c.t_f_gpu},
                {"t_f_ssd_s", c.t_f_ssd},         {"t_f_s", c.t_f},
                {"t_b_comp_s", c.t_b_comp},       {"t_o_comp_s", c.t_o_comp},
                {"t_bo_gpu_s", c.t_bo_gpu},       {"t_bo_gpu_c2g_s", c.t_bo_gpu_c2g},
                {"t_bo_gpu_g2c_s", c.t_bo_gpu_g2c}, {"t_bo_ssd_s", c.t_bo_ssd},
                {"t_bo_s", c.t_bo},               {"t_iter_s", c.t_iter},
                {"d_f_bytes", c.d_f},             {"bottleneck_f", to_string(c.bottleneck_f)},
                {"bottleneck_bo", to_string(c.bottleneck_bo)}};
}

json plan_json(const ModelConfig& model, const SwapPlan& plan) {
    const std::vector<LayerProfile> layers = build_layer_profiles(model);
    json names = json::array();
    for (const std::uint32_t i : plan.swapped_layers) {
        std::ostringstream os;
        os << "b" << layers[i].block_index << " " << to_string(layers[i].kind);
        names.push_back(os.str());
    }
    return json{{"d_start_bytes", plan.d_start_bytes},
                {"d_f_bytes", plan.d_f_bytes},
                {"d_max_bytes", plan.d_max_bytes},
                {"t_max_s", plan.t_max_s},
                {"swap_coefficient", plan.swap_coefficient},
                {"swapped_layer_count", plan.swapped_layers.size()},
                {"swapped_layers", names},
                {"checkpoint_location", plan.checkpoints_on_ssd ? "ssd" : "cpu"}};
}

json echo_json(const Scenario& s) {
    return json{{"model", s.model.name},         {"hardware", s.hardware.name},
                {"batch_size", s.model.batch_size}, {"seq_len", s.model.seq_len},
                {"n_ssd", s.hardware.n_ssd},     {"variant", to_string(s.variant)},
                {"seed", s.seed}};
}

PlannerOptions options_for(const Scenario& s, bool ckpt_on_ssd) {
    PlannerOptions o;
    o.mode = s.planner_mode;
    o.fixed_d_f_bytes = s.planner_value;
    o.fixed_coefficient = s.planner_value;
    o.checkpoints_on_ssd = ckpt_on_ssd;
    return o;
}

} // namespace

bool checkpoints_fit_cpu(const ModelConfig& model, const HardwareConfig& hw) {
    const FootprintReport fp = footprint(model);
    const std::uint64_t everything = fp.total_checkpoint_bytes + total_intra_block_act_bytes(model);
    const std::uint64_t stage = staging_bytes(model);
    return stage <= hw.cpu_mem && everything <= hw.cpu_mem - stage;
}

SwapPlan plan_for_scenario(const Scenario& s) {
    const bool on_ssd =
        s.variant != ScheduleVariant::serial && !checkpoints_fit_cpu(s.model, s.hardware);
    return plan_swaps(s.model, s.hardware, options_for(s, on_ssd));
}

RunOutputs run_scenario(const Scenario& s) {
    RunOutputs r;
    r.plan = plan_for_scenario(s);
    r.graph = build_schedule(s.model, s.hardware, r.plan, s.variant);
    r.trace = simulate(r.graph, s.hardware);
    r.invariants = check_trace_invariants(r.graph, r.trace, s.hardware);
    return r;
}

std::string plan_report_json(const Scenario& s) {
    const SwapPlan plan = plan_for_scenario(s);
    const json doc = {{"schema_version", kScenarioSchemaVersion},
                      {"command", "plan"},
                      {"scenario", echo_json(s)},
                      {"plan", plan_json(s.model, plan)},
                      {"cost_model", breakdown_json(plan.predicted)}};
    return doc.dump(2) + "\n";
}

std::string simulate_summary_json(const Scenario& s, std::string* trace_json_out) {
    const RunOutputs run = run_scenario(s);
    if (trace_json_out) *trace_json_out = to_chrome_trace_json(run.graph, run.trace);
    json busy = json::object();
    for (const auto& [lane, ns] : run.trace.busy_ns) busy[to_string(lane)] = static_cast<double>(ns) * 1e-9;
    json peaks = json::object();
    for (const auto& [pool, bytes] : run.trace.peak_mem) peaks[to_string(pool)] = bytes;
    json checks = json::array();
    for (const auto& e : run.invariants.entries)
        checks.push_back(json{{"name", e.name}, {"pass", e.pass}, {"detail", e.detail}});
    const json sim = {
        {"variant", to_string(s.variant)},
        {"checkpoint_location", run.graph.header.checkpoint_location},
        {"makespan_s", run.trace.makespan_s()},
        {"makespan_ns", run.trace.makespan_ns},
        {"task_count", run.graph.tasks.size()},
        {"peak_mem_bytes", peaks},
        {"busy_s", busy},
        {"roofline_lower_bound_s",
         static_cast<double>(roofline_lower_bound_ns(run.graph, s.hardware)) * 1e-9},
        {"serial_duration_sum_s",
         static_cast<double>(serial_duration_sum_ns(run.graph, s.hardware)) * 1e-9},
    };
    const json doc = {{"schema_version", kScenarioSchemaVersion},
                      {"command", "simulate"},
                      {"scenario", echo_json(s)},
                      {"plan", plan_json(s.model, run.plan)},
                      {"cost_model", breakdown_json(run.plan.predicted)},
                      {"simulation", sim},
                      {"invariants", checks},
                      {"all_invariants_pass", run.invariants.all_pass}};
    return doc.dump(2) + "\n";
}

namespace {

constexpr ScheduleVariant kVariants[] = {ScheduleVariant::serial, ScheduleVariant::pipelined,
                                         ScheduleVariant::overlapped};

Scenario with_axis(const Scenario& base, const std::string& axis, double value) {
    Scenario s = base;
    if (axis == "batch_size") {
        if (value < 1.0) throw ConfigError("batch_size value must be >= 1");
        s.model.batch_size = static_cast<std::uint64_t>(value);
    } else if (axis == "n_ssd") {
        if (value < 1.0) throw ConfigError("n_ssd value must be >= 1");
        s.hardware.n_ssd = static_cast<std::uint32_t>(value);
    } else if (axis == "swap_coefficient") {
        s.planner_mode = PlannerOptions::Mode::fixed_coefficient;
        s.planner_value = value;
    } else if (axis == "cpu_mem") {
        if (value <= 0.0) throw ConfigError("cpu_mem value (GB) must be > 0");
        s.hardware.cpu_mem = static_cast<std::uint64_t>(value * 1e9);
    } else {
        throw ConfigError("unknown sweep axis '" + axis + "'");
    }
    return s;
}

struct Cell {
    std::size_t vi = 0;
    double value = 0.0;
    ScheduleVariant variant = ScheduleVariant::serial;
    bool ok = false;
    std::string error;
    double makespan_s = 0.0;
    SwapPlan plan;
    std::string ckpt_location;
};

void evaluate(const Scenario& base, const std::string& axis, Cell& c) {
    try {
        Scenario s = with_axis(base, axis, c.value);
        s.variant = c.variant;
        const RunOutputs r = run_scenario(s);
        if (!r.invariants.all_pass) {
            c.ok = false;
            c.error = "trace invariant failure";
            return;
        }
        c.ok = true;
        c.makespan_s = r.trace.makespan_s();
        c.plan = r.plan;
        c.ckpt_location = r.graph.header.checkpoint_location;
    } catch (const std::exception& e) {
        c.ok = false;
        c.error = e.what();
    }
}

std::string csv_safe(std::string s) {
    std::replace_if(s.begin(), s.end(), [](char ch) { return ch == ',' || ch == '\n'; }, ';');
    return s;
}

} // namespace

std::string sweep_csv(const Scenario& base, const std::string& axis,
                      const std::vector<double>& values, int workers) {
    if (values.empty()) throw ConfigError("sweep: values list must not be empty");
    if (axis != "batch_size" && axis != "n_ssd" && axis != "swap_coefficient" && axis != "cpu_mem")
        throw ConfigError("unknown sweep axis '" + axis + "'");
    std::vector<Cell> cells;
    for (std::size_t vi = 0; vi < values.size(); ++vi)
        for (const ScheduleVariant v : kVariants) {
            Cell c;
            c.vi = vi;
            c.value = values[vi];
            c.variant = v;
            cells.push_back(c);
        }
    const int nthreads = std::max(1, std::min<int>(workers, static_cast<int>(cells.size())));
    if (nthreads == 1) {
        for (Cell& c : cells) evaluate(base, axis, c);
    } else {
        std::atomic<std::size_t> cursor{0};
        std::vector<std::thread> pool;
        for (int t = 0; t < nthreads; ++t)
            pool.emplace_back([&] {
                for (std::size_t i; (i = cursor.fetch_add(1)) < cells.size();) evaluate(base, axis, cells[i]);
            });
        for (std::thread& t : pool) t.join();
    }

    const PriceTable prices = price_table(base.hardware);
    std::ostringstream out;
    out << "schema_version,axis,value,variant,status,makespan_s,speedup_vs_serial,"
           "t_f_comp_s,t_f_gpu_s,t_f_ssd_s,t_f_s,t_b_comp_s,t_o_comp_s,t_bo_gpu_s,"
           "t_bo_ssd_s,t_bo_s,t_iter_model_s,bottleneck_f,bottleneck_bo,swap_coefficient,"
           "d_f_bytes,checkpoint_location,tokens_per_s,tokens_per_s_per_dollar_gpu_ssd,"
           "tokens_per_s_per_dollar_server,error\n";
    auto find_cell = [&](std::size_t vi, ScheduleVariant v) -> const Cell* {
        const Cell* hit = nullptr;
        for (const Cell& c : cells)
            if (c.vi == vi && c.variant == v) hit = &c;
        return hit;
    };
    for (std::size_t vi = 0; vi < values.size(); ++vi) {
        const Cell* serial = find_cell(vi, ScheduleVariant::serial);
        for (const ScheduleVariant v : kVariants) {
            const Cell* c = find_cell(vi, v);
            out << kScenarioSchemaVersion << ',' << axis << ',' << g9(values[vi]) << ','
                << to_string(v) << ',';
            if (!c->ok) {
                out << "error" << std::string(21, ',') << csv_safe(c->error) << "\n";
                continue;
            }
            const Scenario varied = with_axis(base, axis, values[vi]);
            out << "ok," << g9(c->makespan_s) << ',';
            if (serial && serial->ok && c->makespan_s > 0.0) out << g9(serial->makespan_s / c->makespan_s);
            const CostBreakdown& cb = c->plan.predicted;
            for (const double x : {cb.t_f_comp, cb.t_f_gpu, cb.t_f_ssd, cb.t_f, cb.t_b_comp,
                                   cb.t_o_comp, cb.t_bo_gpu, cb.t_bo_ssd, cb.t_bo, cb.t_iter})
                out << ',' << g9(x);
            out << ',' << to_string(cb.bottleneck_f) << ',' << to_string(cb.bottleneck_bo) << ','
                << g9(c->plan.swap_coefficient) << ',' << c->plan.d_f_bytes << ','
                << c->ckpt_location << ',';
            out << g9(c->makespan_s > 0.0 ? tokens_per_second(varied.model, c->makespan_s) : 0.0)
                << ',';
            const std::uint32_t n_ssd = varied.hardware.n_ssd;
            if (prices.gpu > 0.0 && prices.ssd > 0.0 && c->makespan_s > 0.0)
                out << g9(cost_effectiveness(c->makespan_s, varied.model, prices,
                                             PriceScope::gpu_ssd, n_ssd));
            out << ',';
            if (prices.gpu > 0.0 && prices.ssd > 0.0 && prices.server > 0.0 && c->makespan_s > 0.0)
                out << g9(cost_effectiveness(c->makespan_s, varied.model, prices,
                                             PriceScope::whole_server, n_ssd));
            out << ",\n";
        }
    }
    return out.str();
}

std::string capacity_csv(const Scenario& base, const std::vector<double>& cpu_mem_gb) {
    if (cpu_mem_gb.empty()) throw ConfigError("capacity: cpu_mem list must not be empty");
    std::vector<ModelConfig> ladder = model_ladder();
    for (ModelConfig& m : ladder) {
        m.batch_size = base.model.batch_size;
        m.seq_len = base.model.seq_len;
    }
    std::ostringstream out;
    out << "schema_version,cpu_mem_gb,policy,max_model,max_params,bottleneck\n";
    for (const double gb : cpu_mem_gb) {
        if (gb <= 0.0) throw ConfigError("capacity: cpu_mem values (GB) must be > 0");
        HardwareConfig hw = base.hardware;
        hw.cpu_mem = static_cast<std::uint64_t>(gb * 1e9);
        for (const PolicyId p : {PolicyId::zero_infinity, PolicyId::two_level}) {
            const MaxTrainable mt = max_trainable(p, hw, ladder);
            out << kScenarioSchemaVersion << ',' << g9(gb) << ',' << to_string(p) << ',';
            if (mt.found)
                out << mt.model.name << ',' << total_param_count(mt.model) << ','
                    << to_string(mt.limit) << "\n";
            else
                out << "none,0," << to_string(mt.limit) << "\n";
        }
    }
    return out.str();
}

std::string validate_report_json(const Scenario& s) {
    const ValidationReport r = validate(s.hardware, &s.model);
    const FootprintReport fp = footprint(s.model);
    const json doc = {
        {"schema_version", kScenarioSchemaVersion},
        {"command", "validate"},
        {"scenario", echo_json(s)},
        {"hardware_validation", json{{"errors", r.errors}, {"warnings", r.warnings}}},
        {"model_footprint",
         json{{"total_params", fp.total_params},
              {"fp16_param_bytes", fp.fp16_param_bytes},
              {"fp16_grad_bytes", fp.fp16_grad_bytes},
              {"optimizer_state_bytes", fp.optimizer_state_bytes},
              {"model_state_bytes", fp.model_state_bytes},
              {"checkpoint_bytes_per_block", fp.checkpoint_bytes_per_block},
              {"total_checkpoint_bytes", fp.total_checkpoint_bytes},
              {"gpu_working_set_bytes", gpu_working_set_bytes(s.model)}}},
        {"ok", r.ok()},
    };
    return doc.dump(2) + "\n";
}

} // namespace offsim
