// Discrete-event simulator, trace validator and Chrome-trace export —
// restates proj/src/simulator.cpp, proj/src/trace_checks.cpp and
// proj/src/trace_export.cpp. The DES is the planning-side executor; the
// B200 executor (exec.cpp) produces the same SimTrace type from CUDA events
// and is validated by the same check_trace_invariants.

#include "offsim/errors.hpp"
#include "offsim/sim.hpp"

#include <algorithm>
#include <array>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <queue>
#include <sstream>

namespace offsim {

namespace {

constexpr std::array<ResourceId, 5> kLanes = {ResourceId::gpu_compute, ResourceId::cpu_compute,
                                              ResourceId::link_c2g, ResourceId::link_g2c,
                                              ResourceId::link_ssd};

double lane_rate(const Task& t, const HardwareConfig& hw) {
    switch (t.resource) {
    case ResourceId::gpu_compute: return hw.gpu_tput;
    case ResourceId::cpu_compute: return hw.cpu_opt_tput;
    case ResourceId::link_c2g:
    case ResourceId::link_g2c: return hw.bw_gpu;
    case ResourceId::link_ssd:
        return aggregate_ssd_bw(hw, t.dir == TransferDir::s2c ? SsdDirection::s2c
                                                              : SsdDirection::c2s);
    default: break;
    }
    throw InvariantError("task '" + t.name + "' scheduled on a memory resource");
}

using Key = std::pair<std::uint64_t, std::uint32_t>; // (time, task id)
using MinHeap = std::priority_queue<Key, std::vector<Key>, std::greater<>>;

} // namespace

std::uint64_t task_duration_ns(const Task& task, const HardwareConfig& hw) {
    if (task.work <= 0.0) return 0;
    return static_cast<std::uint64_t>(std::llround(task.work / lane_rate(task, hw) * 1e9));
}

std::uint64_t serial_duration_sum_ns(const TaskGraph& graph, const HardwareConfig& hw) {
    std::uint64_t total = 0;
    for (const Task& t : graph.tasks) total += task_duration_ns(t, hw);
    return total;
}

std::uint64_t roofline_lower_bound_ns(const TaskGraph& graph, const HardwareConfig& hw) {
    std::map<ResourceId, std::uint64_t> per_lane;
    for (const Task& t : graph.tasks) per_lane[t.resource] += task_duration_ns(t, hw);
    std::uint64_t bound = 0;
    for (const auto& kv : per_lane) bound = std::max(bound, kv.second);
    return bound;
}

namespace {

// Capacity-checked memory pools.
class Pools {
public:
    explicit Pools(const HardwareConfig& hw)
        : cap_{{ResourceId::mem_gpu, static_cast<std::int64_t>(hw.gpu_mem)},
               {ResourceId::mem_cpu, static_cast<std::int64_t>(hw.cpu_mem)}} {}

    void seed(const std::map<ResourceId, std::int64_t>& initial) {
        for (const auto& [pool, bytes] : initial) {
            level_[pool] += bytes;
            peak_[pool] = std::max(peak_[pool], level_[pool]);
        }
        for (const auto& [pool, lvl] : level_) {
            const auto c = cap_.find(pool);
            if (c != cap_.end() && lvl > c->second)
                throw InvariantError(std::string("initial ") + to_string(pool) +
                                     " level exceeds capacity");
        }
    }

    void apply(const Task& t, bool at_start, std::uint64_t now) {
        for (const MemEffect& e : t.mem_effects) {
            if (e.at_start != at_start) continue;
            const std::int64_t lvl = (level_[e.mem] += e.delta_bytes);
            peak_[e.mem] = std::max(peak_[e.mem], lvl);
            const auto c = cap_.find(e.mem);
            if (c != cap_.end() && lvl > c->second) {
                std::ostringstream os;
                os << to_string(e.mem) << " capacity " << c->second << " exceeded (" << lvl
                   << " bytes) by task '" << t.name << "' at " << now << " ns";
                throw InvariantError(os.str());
            }
        }
    }

    const std::map<ResourceId, std::int64_t>& peak() const { return peak_; }

private:
    std::map<ResourceId, std::int64_t> cap_, level_, peak_;
};

} // namespace

SimTrace simulate(const TaskGraph& graph, const HardwareConfig& hw) {
    const std::size_t n = graph.tasks.size();
    std::vector<std::uint64_t> dur(n);
    std::vector<std::uint32_t> waiting(n);
    std::vector<std::vector<std::uint32_t>> successors(n);
    for (const Task& t : graph.tasks) {
        dur[t.id] = task_duration_ns(t, hw);
        waiting[t.id] = static_cast<std::uint32_t>(t.deps.size());
        for (const std::uint32_t d : t.deps) {
            if (d >= n) throw InvariantError("task '" + t.name + "' depends on unknown task");
            successors[d].push_back(t.id);
        }
    }

    Pools pools(hw);
    pools.seed(graph.initial_mem);

    // Per lane: ready tasks ordered by (release time, id) and a busy flag.
    std::array<MinHeap, 7> ready;
    std::array<bool, 7> busy{};
    std::array<std::uint64_t, 7> busy_ns{};
    MinHeap finishing; // (end time, id)
    std::vector<std::uint64_t> started(n, 0);
    std::vector<bool> finished(n, false);

    SimTrace trace;
    trace.header = graph.header;
    trace.events.reserve(n);

    auto lane_of = [&](std::uint32_t id) { return static_cast<std::size_t>(graph.tasks[id].resource); };
    auto dispatch = [&](std::uint64_t now) {
        for (const ResourceId lane : kLanes) {
            const auto li = static_cast<std::size_t>(lane);
            if (busy[li] || ready[li].empty()) continue;
            const std::uint32_t id = ready[li].top().second;
            ready[li].pop();
            started[id] = now;
            pools.apply(graph.tasks[id], true, now);
            busy[li] = true;
            finishing.emplace(now + dur[id], id);
        }
    };

    for (std::uint32_t i = 0; i < n; ++i)
        if (waiting[i] == 0) ready[lane_of(i)].emplace(0, i);
    dispatch(0);

    std::size_t done = 0;
    std::uint64_t makespan = 0;
    while (!finishing.empty()) {
        const std::uint64_t now = finishing.top().first;
        // Retire everything ending at `now` before anything starts at `now`,
        // so memory freed at this instant is visible to new starts.
        while (!finishing.empty() && finishing.top().first == now) {
            const std::uint32_t id = finishing.top().second;
            finishing.pop();
            const Task& t = graph.tasks[id];
            finished[id] = true;
            busy[lane_of(id)] = false;
            busy_ns[lane_of(id)] += dur[id];
            pools.apply(t, false, now);
            trace.events.push_back(TraceEvent{id, t.resource, t.dir, t.payload, t.work, started[id], now});
            ++done;
            makespan = std::max(makespan, now);
            for (const std::uint32_t s : successors[id])
                if (--waiting[s] == 0) ready[lane_of(s)].emplace(now, s);
        }
        dispatch(now);
    }

    if (done < n) {
        std::ostringstream os;
        os << "deadlock: " << (n - done) << " tasks blocked, first:";
        int shown = 0;
        for (std::size_t i = 0; i < n && shown < 4; ++i)
            if (!finished[i]) {
                os << " '" << graph.tasks[i].name << "'";
                ++shown;
            }
        throw InvariantError(os.str());
    }

    trace.makespan_ns = makespan;
    trace.peak_mem = pools.peak();
    for (const ResourceId lane : kLanes) trace.busy_ns[lane] = busy_ns[static_cast<std::size_t>(lane)];
    return trace;
}

// ------------------------------------------------------------ validation

namespace {

void record(InvariantReport& r, std::string name, bool pass, std::string detail = "") {
    r.entries.push_back({std::move(name), pass, std::move(detail)});
    r.all_pass = r.all_pass && pass;
}

bool by_start_then_end(const TraceEvent* a, const TraceEvent* b) {
    return a->start_ns != b->start_ns ? a->start_ns < b->start_ns : a->end_ns < b->end_ns;
}

} // namespace

InvariantReport check_trace_invariants(const TaskGraph& graph, const SimTrace& trace,
                                       const HardwareConfig& hw) {
    InvariantReport report;
    const std::size_t n = graph.tasks.size();

    { // every task ran exactly once with end >= start
        bool ok = trace.events.size() == n;
        std::string why;
        std::vector<bool> seen(n, false);
        for (const TraceEvent& e : trace.events) {
            if (e.task_id >= n || seen[e.task_id] || e.end_ns < e.start_ns) {
                ok = false;
                why = "bad event for task " + std::to_string(e.task_id);
                break;
            }
            seen[e.task_id] = true;
        }
        record(report, "all-tasks-executed", ok, why);
    }

    std::vector<const TraceEvent*> ev_of(n, nullptr);
    for (const TraceEvent& e : trace.events)
        if (e.task_id < n) ev_of[e.task_id] = &e;

    { // every task starts after all its dependencies end
        bool ok = true;
        std::string why;
        for (const Task& t : graph.tasks) {
            if (!ok) break;
            if (!ev_of[t.id]) continue;
            for (const std::uint32_t d : t.deps) {
                if (!ev_of[d]) continue;
                if (ev_of[t.id]->start_ns < ev_of[d]->end_ns) {
                    ok = false;
                    why = "task '" + t.name + "' started before its dependency '" +
                          graph.tasks[d].name + "' finished";
                    break;
                }
            }
        }
        record(report, "dependencies-respected", ok, why);
    }

    { // one task at a time per serial lane
        bool ok = true;
        std::string why;
        for (const ResourceId lane : kLanes) {
            std::vector<const TraceEvent*> on_lane;
            for (const TraceEvent& e : trace.events)
                if (e.resource == lane) on_lane.push_back(&e);
            std::sort(on_lane.begin(), on_lane.end(), by_start_then_end);
            for (std::size_t i = 1; i < on_lane.size() && ok; ++i) {
                if (on_lane[i]->start_ns < on_lane[i - 1]->end_ns) {
                    ok = false;
                    why = std::string("overlap on ") + to_string(lane) + ": tasks '" +
                          graph.tasks[on_lane[i - 1]->task_id].name + "' and '" +
                          graph.tasks[on_lane[i]->task_id].name + "'";
                }
            }
            if (!ok) break;
        }
        record(report, "serial-resource-exclusive", ok, why);
    }

    { // pools within capacity at every boundary (ends before starts at a tie)
        bool ok = true;
        std::string why;
        struct Edge {
            std::uint64_t t;
            bool start;
            const TraceEvent* e;
        };
        std::vector<Edge> edges;
        edges.reserve(2 * trace.events.size());
        for (const TraceEvent& e : trace.events) {
            edges.push_back({e.start_ns, true, &e});
            edges.push_back({e.end_ns, false, &e});
        }
        std::stable_sort(edges.begin(), edges.end(), [](const Edge& a, const Edge& b) {
            return a.t != b.t ? a.t < b.t : (!a.start && b.start);
        });
        std::map<ResourceId, std::int64_t> level = graph.initial_mem;
        const std::map<ResourceId, std::int64_t> cap = {
            {ResourceId::mem_gpu, static_cast<std::int64_t>(hw.gpu_mem)},
            {ResourceId::mem_cpu, static_cast<std::int64_t>(hw.cpu_mem)}};
        for (const Edge& ed : edges) {
            const Task& t = graph.tasks[ed.e->task_id];
            for (const MemEffect& fx : t.mem_effects) {
                if (fx.at_start != ed.start) continue;
                level[fx.mem] += fx.delta_bytes;
                const auto c = cap.find(fx.mem);
                if (c != cap.end() && level[fx.mem] > c->second) {
                    ok = false;
                    why = std::string(to_string(fx.mem)) + " exceeds capacity at task '" + t.name + "'";
                }
            }
        }
        if (!trace.header.forward_only) {
            for (const auto& [pool, lvl] : level) {
                const auto init = graph.initial_mem.find(pool);
                const std::int64_t base = init == graph.initial_mem.end() ? 0 : init->second;
                if (lvl != base) {
                    ok = false;
                    why = std::string("memory ") + to_string(pool) +
                          " does not return to its initial level";
                }
            }
        }
        record(report, "memory-within-capacity", ok, why);
    }

    {
        const std::uint64_t bound = roofline_lower_bound_ns(graph, hw);
        std::ostringstream os;
        os << "makespan " << trace.makespan_ns << " ns vs bound " << bound << " ns";
        record(report, "roofline-lower-bound", trace.makespan_ns >= bound, os.str());
    }

    if (trace.header.variant == ScheduleVariant::serial) {
        bool ok = true;
        std::string why;
        std::vector<const TraceEvent*> all;
        for (const TraceEvent& e : trace.events) all.push_back(&e);
        std::sort(all.begin(), all.end(), by_start_then_end);
        for (std::size_t i = 1; i < all.size(); ++i)
            if (all[i]->start_ns < all[i - 1]->end_ns) {
                ok = false;
                why = "tasks overlap in a serial schedule";
                break;
            }
        record(report, "strictly-serial", ok, why);
        const std::uint64_t sum = serial_duration_sum_ns(graph, hw);
        std::ostringstream os;
        os << "makespan " << trace.makespan_ns << " ns vs duration sum " << sum << " ns";
        record(report, "makespan-equals-duration-sum", trace.makespan_ns == sum, os.str());
    }

    {
        double grad_bytes = 0.0;
        for (const TraceEvent& e : trace.events)
            if (e.resource == ResourceId::link_ssd && e.payload == Payload::grads) grad_bytes += e.work;
        if (trace.header.variant == ScheduleVariant::overlapped) {
            std::ostringstream os;
            os << grad_bytes << " gradient bytes on the SSD lane";
            record(report, "no-gradient-bytes-on-ssd", grad_bytes == 0.0, os.str());
        } else if (!trace.header.forward_only) {
            const double expect = 2.0 * static_cast<double>(trace.header.fp16_param_bytes);
            std::ostringstream os;
            os << grad_bytes << " gradient bytes on the SSD lane, expected " << expect;
            record(report, "gradient-ssd-roundtrip", grad_bytes == expect, os.str());
        }
    }
    return report;
}

// ----------------------------------------------------------- chrome trace

namespace {

void put_escaped(std::string& out, const std::string& s) {
    for (const char c : s) {
        if (c == '"') out += "\\\"";
        else if (c == '\\') out += "\\\\";
        else if (c == '\n') out += "\\n";
        else if (c == '\t') out += "\\t";
        else if (static_cast<unsigned char>(c) < 0x20) {
            char buf[8];
            std::snprintf(buf, sizeof buf, "\\u%04x", c);
            out += buf;
        } else {
            out += c;
        }
    }
}

void put_us(std::string& out, std::uint64_t ns) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%" PRIu64 ".%03u", ns / 1000, static_cast<unsigned>(ns % 1000));
    out += buf;
}

} // namespace

std::string to_chrome_trace_json(const TaskGraph& graph, const SimTrace& trace) {
    static const char* const kLaneTitle[] = {"GPU compute", "CPU compute", "CPU to GPU",
                                             "GPU to CPU",  "SSD array",   "GPU memory",
                                             "CPU memory"};
    std::vector<const TraceEvent*> order;
    order.reserve(trace.events.size());
    for (const TraceEvent& e : trace.events) order.push_back(&e);
    std::sort(order.begin(), order.end(), [](const TraceEvent* a, const TraceEvent* b) {
        if (a->start_ns != b->start_ns) return a->start_ns < b->start_ns;
        if (a->resource != b->resource) return a->resource < b->resource;
        return a->task_id < b->task_id;
    });
    std::string out;
    out.reserve(order.size() * 160 + 1024);
    out += "{\"traceEvents\":[\n{\"name\":\"process_name\",\"ph\":\"M\",\"pid\":1,\"tid\":0,\"args\":{\"name\":\"";
    put_escaped(out, graph.header.model_name.empty() ? "offsim" : graph.header.model_name);
    out += " (";
    out += to_string(graph.header.variant);
    out += ")\"}}";
    for (int lane = 0; lane < 5; ++lane) {
        out += ",\n{\"name\":\"thread_name\",\"ph\":\"M\",\"pid\":1,\"tid\":" + std::to_string(lane) +
               ",\"args\":{\"name\":\"";
        put_escaped(out, kLaneTitle[lane]);
        out += "\"}}";
    }
    for (const TraceEvent* e : order) {
        const Task& t = graph.tasks[e->task_id];
        out += ",\n{\"name\":\"";
        put_escaped(out, t.name);
        out += "\",\"cat\":\"";
        out += to_string(t.kind);
        out += "\",\"ph\":\"X\",\"ts\":";
        put_us(out, e->start_ns);
        out += ",\"dur\":";
        put_us(out, e->end_ns - e->start_ns);
        out += ",\"pid\":1,\"tid\":" + std::to_string(static_cast<int>(e->resource)) +
               ",\"args\":{\"payload\":\"";
        out += to_string(e->payload);
        out += "\",\"work\":";
        char buf[40];
        std::snprintf(buf, sizeof buf, "%.17g", e->work);
        out += buf;
        out += "}}";
    }
    out += "\n],\"displayTimeUnit\":\"ms\"}\n";
    return out;
}

} // namespace offsim
