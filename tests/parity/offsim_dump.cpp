// Parity dump driver (test infrastructure).
//
// One source, compiled twice: against the compiled reference core
// (oracle/ref.mk -> oracle/_ref/offsim_dump_ref) and against this repo's
// liboffsim (Makefile -> build/offsim_dump). Both builds include only the
// public offsim C++ headers, so compiling at all is the source-level drop-in
// check; the printed digests are the bit-exact behaviour check.
//
// For every case it prints one line:
//   <case-name> <fnv1a64 of the canonical dump> <short summary>
// The canonical dump serialises every field of SwapPlan (doubles as %a hex
// floats), TraceHeader, every Task (name, kind, lane, direction, payload,
// work, deps, memory effects), the DES SimTrace (every event, peak memory,
// busy time), the invariant report, and per-(resource, payload) byte totals.
// `--full DIR` also writes each canonical dump to DIR/<case>.txt.
//
// Cases: the reference's scenario presets under all three variants, the
// BASELINE.json configurations, and the reference
// acceptance matrix (220 scenarios x 3 variants, seed 20240817; the matrix
// recipe follows proj/tests/acceptance/acceptance_main.cpp:80-151).

#include "offsim/capacity.hpp"
#include "offsim/cost_model.hpp"
#include "offsim/errors.hpp"
#include "offsim/planner.hpp"
#include "offsim/presets.hpp"
#include "offsim/runner.hpp"
#include "offsim/scenario.hpp"
#include "offsim/sim.hpp"
#include "offsim/workload.hpp"

#include <cstdint>
#include <cstdio>
#include <fstream>
#include <functional>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <vector>

using namespace offsim;

namespace {

std::string hx(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%a", v);
    return buf;
}

std::uint64_t fnv1a(const std::string& s) {
    std::uint64_t h = 1469598103934665603ull;
    for (unsigned char c : s) {
        h ^= c;
        h *= 1099511628211ull;
    }
    return h;
}

void dump_breakdown(std::ostream& os, const CostBreakdown& c) {
    os << "pred " << hx(c.t_f_comp) << ' ' << hx(c.t_f_gpu) << ' ' << hx(c.t_f_ssd) << ' '
       << hx(c.t_f) << ' ' << hx(c.t_b_comp) << ' ' << hx(c.t_o_comp) << ' ' << hx(c.t_bo_gpu)
       << ' ' << hx(c.t_bo_gpu_c2g) << ' ' << hx(c.t_bo_gpu_g2c) << ' ' << hx(c.t_bo_ssd) << ' '
       << hx(c.t_bo) << ' ' << hx(c.t_iter) << ' ' << hx(c.d_f) << ' '
       << to_string(c.bottleneck_f) << ' ' << to_string(c.bottleneck_bo) << '\n';
}

void dump_plan(std::ostream& os, const SwapPlan& p) {
    os << "plan " << p.d_start_bytes << ' ' << p.d_f_bytes << ' ' << hx(p.d_max_bytes) << ' '
       << hx(p.t_max_s) << ' ' << hx(p.swap_coefficient) << ' ' << p.checkpoints_on_ssd
       << " n=" << p.swapped_layers.size() << " [";
    for (auto i : p.swapped_layers) os << i << ',';
    os << "]\n";
    dump_breakdown(os, p.predicted);
}

void dump_graph(std::ostream& os, const TaskGraph& g) {
    const TraceHeader& h = g.header;
    os << "header " << to_string(h.variant) << ' ' << h.model_name << ' ' << h.hardware_name
       << ' ' << h.checkpoint_location << ' ' << h.fp16_param_bytes << ' ' << h.gpu_fifo_bytes
       << ' ' << h.prefetch_window_layers << ' ' << h.offload_window_blocks << ' '
       << h.cpu_stage_window_layers << ' ' << h.forward_only << '\n';
    for (const auto& [r, b] : g.initial_mem) os << "init " << to_string(r) << ' ' << b << '\n';
    for (const Task& t : g.tasks) {
        os << "task " << t.id << " '" << t.name << "' " << to_string(t.kind) << ' '
           << to_string(t.resource) << ' ' << to_string(t.dir) << ' ' << to_string(t.payload)
           << ' ' << hx(t.work) << " d[";
        for (auto d : t.deps) os << d << ',';
        os << "] fx[";
        for (const MemEffect& e : t.mem_effects)
            os << to_string(e.mem) << ':' << e.delta_bytes << ':' << e.at_start << ',';
        os << "]\n";
    }
}

void dump_trace(std::ostream& os, const SimTrace& tr) {
    os << "makespan " << tr.makespan_ns << '\n';
    for (const TraceEvent& e : tr.events)
        os << "ev " << e.task_id << ' ' << to_string(e.resource) << ' ' << to_string(e.dir) << ' '
           << to_string(e.payload) << ' ' << hx(e.work) << ' ' << e.start_ns << ' ' << e.end_ns
           << '\n';
    for (const auto& [r, b] : tr.peak_mem) os << "peak " << to_string(r) << ' ' << b << '\n';
    for (const auto& [r, b] : tr.busy_ns) os << "busy " << to_string(r) << ' ' << b << '\n';
}

void dump_bytes(std::ostream& os, const TaskGraph& g) {
    std::map<std::string, double> sums;
    for (const Task& t : g.tasks)
        if (t.kind == TaskKind::transfer)
            sums[std::string(to_string(t.resource)) + '/' + to_string(t.payload)] += t.work;
    for (const auto& [k, v] : sums) os << "bytes " << k << ' ' << hx(v) << '\n';
}

void dump_invariants(std::ostream& os, const InvariantReport& r) {
    for (const auto& e : r.entries) os << "inv " << e.name << ' ' << e.pass << " " << e.detail << '\n';
    os << "all_pass " << r.all_pass << '\n';
}

struct Case {
    std::string name;
    std::function<void(std::ostream&)> body;
};

// Runs the body, converting library exceptions into a canonical line so
// that error type and message are part of the digest.
std::string run_case(const Case& c) {
    std::ostringstream os;
    try {
        c.body(os);
    } catch (const InfeasibleError& e) {
        os << "error infeasible " << e.what() << '\n';
    } catch (const ConfigError& e) {
        os << "error config " << e.what() << '\n';
    } catch (const InvariantError& e) {
        os << "error invariant " << e.what() << '\n';
    } catch (const std::exception& e) {
        os << "error other " << e.what() << '\n';
    }
    return os.str();
}

void run_full(std::ostream& os, const ModelConfig& m, const HardwareConfig& hw,
              const SwapPlan& plan, ScheduleVariant v) {
    dump_plan(os, plan);
    const TaskGraph g = build_schedule(m, hw, plan, v);
    dump_graph(os, g);
    dump_bytes(os, g);
    const SimTrace tr = simulate(g, hw);
    dump_trace(os, tr);
    os << "roofline " << roofline_lower_bound_ns(g, hw) << " serial_sum "
       << serial_duration_sum_ns(g, hw) << '\n';
    dump_invariants(os, check_trace_invariants(g, tr, hw));
}

ModelConfig shape(const char* name, std::uint32_t l, std::uint32_t heads, std::uint64_t h,
                  std::uint64_t b, std::uint64_t s) {
    ModelConfig m;
    m.name = name;
    m.num_layers = l;
    m.num_heads = heads;
    m.hidden_dim = h;
    m.batch_size = b;
    m.seq_len = s;
    return m;
}

// Acceptance matrix recipe (proj/tests/acceptance/acceptance_main.cpp:80-151).
std::vector<std::pair<ModelConfig, HardwareConfig>> acceptance_matrix() {
    std::mt19937 rng(20240817);
    auto pick = [&rng](const auto& options) {
        std::uniform_int_distribution<std::size_t> d(0, options.size() - 1);
        return options[d(rng)];
    };
    const std::vector<double> bw_gpu = {8e9, 16e9, 25e9, 32e9};
    const std::vector<double> bw_read = {2e9, 4e9, 6e9, 7e9};
    const std::vector<std::uint32_t> ssds = {1, 2, 4, 6, 8, 12};
    const std::vector<double> gpu_tputs = {5e13, 1e14, 1.64e14, 2e14};
    const std::vector<double> opt_tputs = {5e8, 1e9, 2e9, 4e9};
    std::vector<std::pair<ModelConfig, HardwareConfig>> out;
    auto hw_for = [&](const ModelConfig& m) {
        HardwareConfig hw;
        hw.name = "matrix";
        hw.bw_gpu = pick(bw_gpu);
        hw.bw_s2c = pick(bw_read);
        hw.bw_c2s = hw.bw_s2c / 2.0;
        hw.n_ssd = pick(ssds);
        hw.gpu_tput = pick(gpu_tputs);
        hw.cpu_opt_tput = pick(opt_tputs);
        const std::uint64_t ws = gpu_working_set_bytes(m);
        hw.gpu_mem = ws + std::max<std::uint64_t>(ws, 16ull * 1000 * 1000 * 1000);
        const FootprintReport fp = footprint(m);
        const std::uint64_t full_swap = fp.total_checkpoint_bytes + total_intra_block_act_bytes(m);
        const double block_fp16 =
            12.0 * static_cast<double>(m.hidden_dim) * static_cast<double>(m.hidden_dim) * 2.0;
        const auto staging = static_cast<std::uint64_t>(kCpuStagingGroups * block_fp16 * 8.0);
        hw.cpu_mem = (full_swap + staging + fp.fp16_grad_bytes) * 3 / 2 + (1ull << 30);
        hw.ssd_capacity = 1ull << 50;
        return hw;
    };
    const std::vector<std::uint64_t> small_h = {512, 1024, 2048};
    const std::vector<std::uint64_t> small_b = {1, 2, 4, 8};
    const std::vector<std::uint64_t> small_s = {128, 256};
    std::uniform_int_distribution<std::uint32_t> small_blocks(1, 3);
    for (int i = 0; i < 60; ++i) {
        ModelConfig m;
        m.name = "small-" + std::to_string(i);
        m.num_layers = small_blocks(rng);
        m.num_heads = 4;
        m.hidden_dim = pick(small_h);
        m.batch_size = pick(small_b);
        m.seq_len = pick(small_s);
        HardwareConfig hw = hw_for(m);
        out.emplace_back(m, hw);
    }
    const std::vector<std::uint64_t> large_h = {2048, 3072, 4096, 5120, 6144, 8192};
    const std::vector<std::uint64_t> large_b = {1, 2, 4, 8, 16, 32, 48};
    const std::vector<std::uint64_t> large_s = {512, 1024};
    std::uniform_int_distribution<std::uint32_t> large_blocks(8, 96);
    for (int i = 0; i < 160; ++i) {
        ModelConfig m;
        m.name = "large-" + std::to_string(i);
        m.num_layers = large_blocks(rng);
        m.num_heads = 8;
        m.hidden_dim = pick(large_h);
        m.batch_size = pick(large_b);
        m.seq_len = pick(large_s);
        HardwareConfig hw = hw_for(m);
        out.emplace_back(m, hw);
    }
    return out;
}

std::vector<Case> all_cases(bool with_matrix) {
    std::vector<Case> cases;
    const ScheduleVariant variants[3] = {ScheduleVariant::serial, ScheduleVariant::pipelined,
                                         ScheduleVariant::overlapped};

    // Scenario presets through the orchestration layer (runner) and the
    // report JSON the C ABI returns.
    for (const std::string& name : scenario_preset_names()) {
        for (ScheduleVariant v : variants) {
            cases.push_back({"preset/" + name + "/" + to_string(v), [name, v](std::ostream& os) {
                                 Scenario s = scenario_preset(name);
                                 s.variant = v;
                                 os << "fit_cpu " << checkpoints_fit_cpu(s.model, s.hardware) << '\n';
                                 const RunOutputs r = run_scenario(s);
                                 dump_plan(os, r.plan);
                                 dump_graph(os, r.graph);
                                 dump_bytes(os, r.graph);
                                 dump_trace(os, r.trace);
                                 dump_invariants(os, r.invariants);
                                 os << plan_report_json(s);
                                 os << simulate_summary_json(s, nullptr);
                                 os << scenario_to_json(s);
                             }});
        }
    }

    // BASELINE.json configurations on the a100-12ssd preset.
    struct Cfg {
        std::string tag;
        ModelConfig m;
    };
    std::vector<Cfg> cfgs = {
        {"C1-gpt2-b8", shape("gpt2-small-shape", 12, 12, 768, 8, 1024)},
        {"C1-gpt2-b128", shape("gpt2-small-shape", 12, 12, 768, 128, 1024)},
        {"C2-13b-b32", shape("gpt3-13b", 40, 40, 5120, 32, 1024)},
        {"C3-65b-b16", shape("gpt3-65b", 80, 64, 8192, 16, 1024)},
        {"C4-175b-b16", shape("gpt3-175b", 96, 96, 12288, 16, 1024)},
    };
    for (std::uint64_t b : {8, 16, 32, 64})
        cfgs.push_back({"C5-13b-s2048-b" + std::to_string(b),
                        shape("gpt3-13b", 40, 40, 5120, b, 2048)});
    for (const Cfg& c : cfgs) {
        for (ScheduleVariant v : variants) {
            cases.push_back({"cfg/" + c.tag + "/" + to_string(v), [c, v](std::ostream& os) {
                                 Scenario s;
                                 s.model = c.m;
                                 s.hardware = hardware_preset("a100-12ssd");
                                 s.variant = v;
                                 os << "fit_cpu " << checkpoints_fit_cpu(s.model, s.hardware) << '\n';
                                 const RunOutputs r = run_scenario(s);
                                 dump_plan(os, r.plan);
                                 dump_graph(os, r.graph);
                                 dump_bytes(os, r.graph);
                                 dump_trace(os, r.trace);
                                 dump_invariants(os, r.invariants);
                             }});
        }
        // Forced SSD placement exercises the GPU->host->SSD leg (C5).
        cases.push_back({"cfg/" + c.tag + "/overlapped-ssd", [c](std::ostream& os) {
                             const HardwareConfig hw = hardware_preset("a100-12ssd");
                             PlannerOptions o;
                             o.checkpoints_on_ssd = true;
                             run_full(os, c.m, hw, plan_swaps(c.m, hw, o),
                                      ScheduleVariant::overlapped);
                         }});
    }

    // Planner modes on the 13B preset.
    for (double coef : {0.0, 0.25, 1.0 / 3.0, 0.5, 1.0}) {
        cases.push_back({"mode/coef-" + hx(coef), [coef](std::ostream& os) {
                             const ModelConfig m = shape("gpt3-13b", 40, 40, 5120, 32, 1024);
                             const HardwareConfig hw = hardware_preset("rtx4090-12ssd");
                             PlannerOptions o;
                             o.mode = PlannerOptions::Mode::fixed_coefficient;
                             o.fixed_coefficient = coef;
                             run_full(os, m, hw, plan_swaps(m, hw, o), ScheduleVariant::overlapped);
                         }});
    }
    for (double df : {0.0, 1e10, 5e10, 2e11}) {
        cases.push_back({"mode/df-" + hx(df), [df](std::ostream& os) {
                             const ModelConfig m = shape("gpt3-13b", 40, 40, 5120, 64, 1024);
                             const HardwareConfig hw = hardware_preset("a100-12ssd");
                             PlannerOptions o;
                             o.mode = PlannerOptions::Mode::fixed_d_f;
                             o.fixed_d_f_bytes = df;
                             run_full(os, m, hw, plan_swaps(m, hw, o), ScheduleVariant::pipelined);
                         }});
    }

    if (with_matrix) {
        const auto matrix = acceptance_matrix();
        for (const auto& [m, hw] : matrix) {
            for (ScheduleVariant v : variants) {
                cases.push_back(
                    {"matrix/" + m.name + "/" + to_string(v), [m = m, hw = hw, v](std::ostream& os) {
                         Scenario s;
                         s.model = m;
                         s.hardware = hw;
                         s.variant = v;
                         os << "fit_cpu " << checkpoints_fit_cpu(m, hw) << '\n';
                         const RunOutputs r = run_scenario(s);
                         dump_plan(os, r.plan);
                         dump_graph(os, r.graph);
                         dump_trace(os, r.trace);
                         dump_invariants(os, r.invariants);
                     }});
            }
        }
    }
    return cases;
}

} // namespace

int main(int argc, char** argv) {
    std::string full_dir;
    bool with_matrix = true;
    std::string only;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--full" && i + 1 < argc) full_dir = argv[++i];
        else if (a == "--no-matrix") with_matrix = false;
        else if (a == "--only" && i + 1 < argc) only = argv[++i];
    }
    for (const Case& c : all_cases(with_matrix)) {
        if (!only.empty() && c.name.find(only) == std::string::npos) continue;
        const std::string text = run_case(c);
        // Summary: first "plan" line's d_f and swapped count, or the error.
        std::string summary;
        std::istringstream is(text);
        for (std::string line; std::getline(is, line);) {
            if (line.rfind("plan ", 0) == 0 || line.rfind("error ", 0) == 0) {
                summary = line.substr(0, 120);
                break;
            }
        }
        std::printf("%s %016llx %s\n", c.name.c_str(), static_cast<unsigned long long>(fnv1a(text)),
                    summary.c_str());
        if (!full_dir.empty()) {
            std::string fn = c.name;
            for (char& ch : fn)
                if (ch == '/') ch = '_';
            std::ofstream(full_dir + "/" + fn + ".txt") << text;
        }
    }
    return 0;
}
