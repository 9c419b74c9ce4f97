// Tier map: rewrites a reference TaskGraph into the graph the B200 executor
// runs (see include/offsim/exec.hpp). Pure graph transformation — testable
// without a GPU (tests/test_tier_map.py through offsim_execute's dry run).
//
// Rules (reference anchors are proj/src/task_graph.cpp lines):
//  * optimizer on the GPU (opt update gK, :488-495): insert
//      "opt state_h2d gK"  link_c2g, 12N B, after state_s2c, before update
//      "opt state_d2h gK"  link_g2c, 12N B, after update, before state_c2s
//      "opt param_d2h gK"  link_g2c,  2N B, after update, before param_c2s
//    (and for serial/pipelined, "opt grad_h2d gK" link_c2g 2N B after
//    grad_s2c: those variants stage gradients through the SSD by definition)
//  * overlapped: grads never leave HBM — bwd grad_g2c (:442-445) moves 0 B
//  * tier host: every link_ssd task moves 0 B (pinned host DRAM is the
//    tier); tier file: link_ssd tasks are real file reads / writes
//  * memory pools re-booked: grad / param bytes leave the GPU pool at
//    param_d2h instead of grad_g2c; the update has no CPU-side effect;
//    states occupy a GPU staging slot from state_h2d to state_d2h.

#include "offsim/errors.hpp"
#include "offsim/exec.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <vector>
#include <string>

namespace offsim {

const char* to_string(StateTier t) { return t == StateTier::host ? "host" : "file"; }

namespace {

bool starts_with(const std::string& s, const char* p) { return s.rfind(p, 0) == 0; }

// "opt update g7" -> "g7"
std::string group_of(const std::string& name) { return name.substr(name.rfind(' ') + 1); }

} // namespace

TaskGraph map_graph_for_b200(const TaskGraph& in, StateTier tier, std::uint32_t state_slots,
                             std::uint32_t resident_groups) {
    if (state_slots < 2) throw ConfigError("executor: state_slots must be >= 2");
    const bool overlapped = in.header.variant == ScheduleVariant::overlapped;
    if (!overlapped && tier == StateTier::host)
        throw ConfigError(std::string("variant '") + to_string(in.header.variant) +
                          "' stages gradients through the SSD; execute it with tier=file");

    TaskGraph out;
    out.header = in.header;
    out.initial_mem = in.initial_mem;
    std::vector<std::uint32_t> remap(in.tasks.size());
    // Per optimizer group: ids of the inserted hops (in the output graph).
    std::map<std::string, std::uint32_t> h2d_of, d2h_of, pd2h_of, gh2d_of;
    // Device staging slot of the m-th optimizer group is m % state_slots; its
    // state_h2d waits for the state_d2h of group m - state_slots (the slot's
    // previous user) — a physical constraint made explicit as a graph edge.
    std::vector<std::uint32_t> d2h_in_order;

    auto push = [&](Task t) {
        t.id = static_cast<std::uint32_t>(out.tasks.size());
        std::sort(t.deps.begin(), t.deps.end());
        t.deps.erase(std::unique(t.deps.begin(), t.deps.end()), t.deps.end());
        out.tasks.push_back(std::move(t));
        return out.tasks.back().id;
    };
    auto hop = [&](const std::string& name, ResourceId lane, TransferDir dir, Payload p,
                   double bytes, std::vector<std::uint32_t> deps, std::vector<MemEffect> fx) {
        Task t;
        t.name = name;
        t.kind = TaskKind::transfer;
        t.resource = lane;
        t.dir = dir;
        t.payload = p;
        t.work = bytes;
        t.deps = std::move(deps);
        t.mem_effects = std::move(fx);
        return push(std::move(t));
    };

    // Pass 1: block geometry from the reference's own tasks.
    std::map<std::string, double> state_bytes, param_bytes;
    for (const Task& t : in.tasks) {
        if (starts_with(t.name, "opt state_s2c ")) state_bytes[group_of(t.name)] = t.work;
        if (starts_with(t.name, "opt param_c2s ")) param_bytes[group_of(t.name)] = t.work;
    }
    // groups "g0".."g(R-1)" keep their states in HBM for the whole run
    auto resident = [&](const std::string& g) {
        return resident_groups > 0 && g.size() > 1 && g[0] == 'g' &&
               std::stoul(g.substr(1)) < resident_groups;
    };
    for (const auto& [g, sb] : state_bytes)
        if (resident(g)) out.initial_mem[ResourceId::mem_gpu] += static_cast<std::int64_t>(sb);

    for (const Task& src : in.tasks) {
        Task t = src;
        for (auto& d : t.deps) d = remap[d];
        const std::string g = group_of(src.name);
        const auto i64 = [](double b) { return static_cast<std::int64_t>(b); };

        if (t.resource == ResourceId::link_ssd && tier == StateTier::host) t.work = 0.0;
        if ((starts_with(src.name, "opt state_s2c ") || starts_with(src.name, "opt state_c2s ")) && resident(g)) {
            t.work = 0.0;  // resident states never leave HBM
            t.mem_effects.clear();
        }

        if (starts_with(src.name, "bwd grad_g2c ") && overlapped) {
            // gradients stay in HBM and feed the fused kernel directly
            t.work = 0.0;
            t.mem_effects.clear();
        } else if (starts_with(src.name, "opt update ")) {
            if (!overlapped) {
                // grad_s2c landed the grads in CPU memory; bring them back
                // to the device (real bytes, the variant's definition)
                std::uint32_t gs = 0;
                for (const std::uint32_t d : t.deps)
                    if (starts_with(out.tasks[d].name, "opt grad_s2c ")) gs = d;
                const double gb = param_bytes[g];
                gh2d_of[g] = hop("opt grad_h2d " + g, ResourceId::link_c2g, TransferDir::c2g,
                                 Payload::grads, gb, {gs},
                                 {MemEffect{ResourceId::mem_gpu, i64(gb), true},
                                  MemEffect{ResourceId::mem_cpu, -i64(gb), false}});
                t.deps.push_back(gh2d_of[g]);
            }
            // the states go to a device staging slot first
            std::uint32_t state_read = 0;
            for (const std::uint32_t d : t.deps)
                if (starts_with(out.tasks[d].name, "opt state_s2c ")) state_read = d;
            const double sb = state_bytes[g];
            std::vector<std::uint32_t> h2d_deps{state_read};
            if (d2h_in_order.size() >= state_slots)
                h2d_deps.push_back(d2h_in_order[d2h_in_order.size() - state_slots]);
            const bool res = resident(g);
            h2d_of[g] = hop("opt state_h2d " + g, ResourceId::link_c2g, TransferDir::c2g,
                            Payload::opt_states, res ? 0.0 : sb, std::move(h2d_deps),
                            res ? std::vector<MemEffect>{}
                                : std::vector<MemEffect>{MemEffect{ResourceId::mem_gpu, i64(sb), true}});
            t.deps.push_back(h2d_of[g]);
            t.mem_effects.clear();
            const std::uint32_t upd = push(std::move(t));
            remap[src.id] = upd;
            const double pb = param_bytes[g];
            d2h_of[g] = hop("opt state_d2h " + g, ResourceId::link_g2c, TransferDir::g2c,
                            Payload::opt_states, res ? 0.0 : sb, {upd},
                            res ? std::vector<MemEffect>{}
                                : std::vector<MemEffect>{MemEffect{ResourceId::mem_gpu, -i64(sb), false}});
            d2h_in_order.push_back(d2h_of[g]);
            pd2h_of[g] = hop("opt param_d2h " + g, ResourceId::link_g2c, TransferDir::g2c,
                             Payload::params, pb, {upd},
                             {MemEffect{ResourceId::mem_cpu, i64(pb), true},
                              MemEffect{ResourceId::mem_gpu, -i64(pb), false}});
            continue;
        } else if (starts_with(src.name, "opt state_c2s ")) {
            t.deps.push_back(d2h_of.at(g));
        } else if (starts_with(src.name, "opt param_c2s ")) {
            t.deps.push_back(pd2h_of.at(g));
        }
        // serial / pipelined bwd grad_g2c stays a real D2H of the grads
        remap[src.id] = push(std::move(t));
    }
    if (in.header.variant == ScheduleVariant::serial) {
        // keep the serial variant fully chained, inserted hops included
        // (task_graph.cpp:92 chains every task to its predecessor)
        for (Task& t : out.tasks)
            if (t.id > 0 && std::find(t.deps.begin(), t.deps.end(), t.id - 1) == t.deps.end()) {
                t.deps.push_back(t.id - 1);
                std::sort(t.deps.begin(), t.deps.end());
            }
    }
    return out;
}

namespace {

struct RingUse {
    std::uint32_t first, last;
};
struct RingUses {
    std::vector<RingUse> states, params, weights, acts;
};

// Uses of each staging ring in task id order: (first task, last task).
RingUses ring_uses(const TaskGraph& g) {
    std::map<std::string, std::uint32_t> by_name;
    for (const Task& t : g.tasks) by_name[t.name] = t.id;
    const bool acts_on_ssd = g.header.checkpoint_location == "ssd";
    auto partner = [&](const std::string& name, const char* from, const char* to) {
        std::string other = name;
        other.replace(other.find(from), std::strlen(from), to);
        const auto it = by_name.find(other);
        return it == by_name.end() ? 0xffffffffu : it->second;
    };
    RingUses u;
    for (const Task& t : g.tasks) {
        const std::string& n = t.name;
        if (starts_with(n, "opt state_s2c ")) u.states.push_back({t.id, partner(n, "state_s2c", "state_c2s")});
        else if (starts_with(n, "opt param_d2h ")) u.params.push_back({t.id, partner(n, "param_d2h", "param_c2s")});
        else if (n.find(" p_s2c ") != std::string::npos) u.weights.push_back({t.id, partner(n, "p_s2c", "p_c2g")});
        else if (acts_on_ssd && (starts_with(n, "fwd act_g2c ") || starts_with(n, "fwd ckpt_g2c ")))
            u.acts.push_back({t.id, partner(n, "_g2c", "_c2s")});
        else if (acts_on_ssd && (starts_with(n, "bwd act_s2c ") || starts_with(n, "bwd ckpt_s2c ")))
            u.acts.push_back({t.id, partner(n, "_s2c", "_c2g")});
    }
    return u;
}

} // namespace

void add_host_ring_edges(TaskGraph& g, const RingDepths& depths) {
    RingUses u = ring_uses(g);
    const std::pair<std::vector<RingUse>*, std::uint32_t> rings[] = {
        {&u.states, depths.states}, {&u.params, depths.params},
        {&u.weights, depths.weights}, {&u.acts, depths.acts}};
    for (const auto& [uses, slots] : rings) {
        if (slots == 0) continue;
        for (std::size_t k = slots; k < uses->size(); ++k) {
            const RingUse& prev = (*uses)[k - slots];
            if (prev.last == 0xffffffffu) throw InvariantError("host ring: unpaired task '" + g.tasks[prev.first].name + "'");
            Task& t = g.tasks[(*uses)[k].first];
            if (prev.last >= t.id) throw InvariantError("host ring edge would not be topological at '" + t.name + "'");
            t.deps.push_back(prev.last);
            std::sort(t.deps.begin(), t.deps.end());
            t.deps.erase(std::unique(t.deps.begin(), t.deps.end()), t.deps.end());
        }
    }
}

void add_host_ring_edges(TaskGraph& g, std::uint32_t slots) {
    add_host_ring_edges(g, RingDepths{slots, slots, slots, slots});
}

RingDepths host_ring_depths(const TaskGraph& g, const ExecOptions& o) {
    if (o.tier != StateTier::file || (o.host_ring == 0 && !o.host_ring_auto)) return {};
    if (!o.host_ring_auto) return RingDepths{o.host_ring, o.host_ring, o.host_ring, o.host_ring};
    const RingUses u = ring_uses(g);
    auto clamp = [](std::uint64_t want, std::size_t uses) {
        if (uses == 0) return 0u;
        return static_cast<std::uint32_t>(std::min<std::uint64_t>(std::max<std::uint64_t>(want, 2), uses));
    };
    const TraceHeader& h = g.header;
    // activation units per block: the checkpoint plus the swapped linears
    std::uint64_t blocks = 0;
    for (const Task& t : g.tasks)
        if (starts_with(t.name, "fwd ckpt_g2c ")) ++blocks;
    const std::uint64_t act_units = blocks ? (u.acts.size() / 2 + blocks - 1) / blocks : 1;
    RingDepths d;
    d.states = clamp(o.state_slots, u.states.size());
    d.params = clamp(o.state_slots, u.params.size());
    d.weights = clamp((h.cpu_stage_window_layers + 3) / 4, u.weights.size());
    d.acts = clamp(static_cast<std::uint64_t>(h.offload_window_blocks) * act_units, u.acts.size());
    return d;
}

TaskGraph swap_subgraph(const TaskGraph& in, std::uint32_t max_blocks) {
    TaskGraph out;
    out.header = in.header;
    out.initial_mem = in.initial_mem;
    std::vector<std::uint32_t> remap(in.tasks.size(), 0xffffffffu);
    for (const Task& src : in.tasks) {
        if (src.payload != Payload::activations) continue;
        // names: "<phase> <what> b<k>[ <kind>]"
        const std::size_t b = src.name.find(" b", src.name.find(' ') + 1);
        const std::uint32_t blk = static_cast<std::uint32_t>(std::stoul(src.name.substr(b + 2)));
        if (max_blocks && blk >= max_blocks) continue;
        Task t = src;
        t.id = static_cast<std::uint32_t>(out.tasks.size());
        t.deps.clear();
        for (const std::uint32_t d : src.deps)
            if (remap[d] != 0xffffffffu) t.deps.push_back(remap[d]);
        remap[src.id] = t.id;
        out.tasks.push_back(std::move(t));
    }
    return out;
}

HardwareConfig b200_hardware(const HardwareConfig& planned_on, const MeasuredRates& r) {
    // Rates are upper bounds of what the engines delivered (measured burst
    // x 1.05), so the unchanged roofline-lower-bound check stays a valid
    // necessary condition on the real trace.
    HardwareConfig hw = planned_on;
    hw.name = "b200-measured";
    const double head = 1.05;
    hw.bw_gpu = std::max(r.h2d_bps, r.d2h_bps) * head;
    hw.n_ssd = 1;
    // file IO through a virtio / NVMe device cache varies more than copy
    // engines do: wider headroom keeps the bound a valid necessary condition
    const double io_head = 1.5;
    hw.bw_s2c = r.file_read_bps > 0 ? r.file_read_bps * io_head : 1e15;
    hw.bw_c2s = r.file_write_bps > 0 ? r.file_write_bps * io_head : 1e15;
    hw.cpu_opt_tput = r.optimizer_params_per_s * head;
    hw.gpu_tput = r.compute_flops;
    if (r.gpu_mem) hw.gpu_mem = r.gpu_mem;
    if (r.cpu_mem) hw.cpu_mem = r.cpu_mem;
    return hw;
}

HardwareConfig b200_hardware_effective(const HardwareConfig& planned_on, const MeasuredRates& r) {
    HardwareConfig hw = b200_hardware(planned_on, r);
    hw.name = "b200-effective";
    // per direction: the graph's own copies replayed alone (simplex) and
    // with the other direction running (duplex), blended per byte by the
    // share of the lane's planned busy time the other direction overlaps
    auto blend = [](double simplex, double duplex, double burst, double f) {
        if (simplex <= 0) simplex = duplex > 0 ? duplex : burst;
        if (duplex <= 0) duplex = simplex;
        f = std::clamp(f, 0.0, 1.0);
        return 1.0 / ((1.0 - f) / simplex + f / duplex);
    };
    const double up = blend(r.h2d_simplex_effective_bps, r.h2d_effective_bps, r.h2d_bps, r.c2g_overlap);
    const double down = blend(r.d2h_simplex_effective_bps, r.d2h_effective_bps, r.d2h_bps, r.g2c_overlap);
    // one bw_gpu serves both link lanes in the reference's model
    // (simulator.cpp:17-35): the rate of the lane that carries more bytes
    // (the binding one; the other lane then finishes early either way)
    hw.bw_gpu = r.c2g_bytes >= r.g2c_bytes ? up : down;
    if (r.c2g_bytes <= 0 && r.g2c_bytes <= 0) hw.bw_gpu = std::min(up, down);
    // file lane: its requests replayed alone and under copy-engine load,
    // blended the same way by the share of its planned busy time a link
    // lane overlaps
    if (r.file_read_bps > 0)
        hw.bw_s2c = blend(r.file_read_effective_bps, r.file_read_loaded_bps, r.file_read_bps, r.ssd_link_overlap);
    if (r.file_write_bps > 0)
        hw.bw_c2s = blend(r.file_write_effective_bps, r.file_write_loaded_bps, r.file_write_bps, r.ssd_link_overlap);
    hw.cpu_opt_tput = r.optimizer_params_per_s;
    hw.gpu_tput = r.compute_effective_flops > 0 ? r.compute_effective_flops : r.compute_flops / r.compute_headroom;
    return hw;
}

} // namespace offsim

namespace offsim {

AnalyticTimes analytic_iteration(const TaskGraph& mapped, const HardwareConfig& hw) {
    // per phase, per lane: the summed durations the DES would charge
    std::map<ResourceId, std::uint64_t> fwd, bwd;
    for (const Task& t : mapped.tasks) {
        const bool forward = t.name.rfind("fwd ", 0) == 0;
        (forward ? fwd : bwd)[t.resource] += task_duration_ns(t, hw);
    }
    auto busiest = [](const std::map<ResourceId, std::uint64_t>& m, std::string& lane) {
        std::uint64_t best = 0;
        for (const auto& [r, ns] : m)
            if (ns > best) {
                best = ns;
                lane = to_string(r);
            }
        return static_cast<double>(best) * 1e-9;
    };
    AnalyticTimes a;
    a.t_f = busiest(fwd, a.bottleneck_f);
    a.t_bo = busiest(bwd, a.bottleneck_bo);
    a.t_iter = a.t_f + a.t_bo;
    return a;
}

} // namespace offsim

namespace offsim {

void link_overlap(const TaskGraph& graph, const SimTrace& trace, MeasuredRates& r) {
    // busy intervals per link lane (a lane is serial: its events do not overlap)
    std::vector<std::pair<std::uint64_t, std::uint64_t>> up, down, ssd, link;
    double ub = 0, db = 0;
    for (const TraceEvent& e : trace.events) {
        if (e.end_ns <= e.start_ns) continue;
        if (e.resource == ResourceId::link_ssd) ssd.emplace_back(e.start_ns, e.end_ns);
        if (e.resource == ResourceId::link_c2g || e.resource == ResourceId::link_g2c)
            link.emplace_back(e.start_ns, e.end_ns);
        if (e.resource == ResourceId::link_c2g) {
            up.emplace_back(e.start_ns, e.end_ns);
            ub += graph.tasks[e.task_id].work;
        } else if (e.resource == ResourceId::link_g2c) {
            down.emplace_back(e.start_ns, e.end_ns);
            db += graph.tasks[e.task_id].work;
        }
    }
    std::sort(up.begin(), up.end());
    std::sort(down.begin(), down.end());
    auto total = [](const std::vector<std::pair<std::uint64_t, std::uint64_t>>& v) {
        double t = 0;
        for (const auto& [a, b] : v) t += static_cast<double>(b - a);
        return t;
    };
    double both = 0;
    for (std::size_t i = 0, j = 0; i < up.size() && j < down.size();) {
        const std::uint64_t lo = std::max(up[i].first, down[j].first);
        const std::uint64_t hi = std::min(up[i].second, down[j].second);
        if (hi > lo) both += static_cast<double>(hi - lo);
        if (up[i].second < down[j].second) ++i;
        else ++j;
    }
    const double tu = total(up), td = total(down);
    r.c2g_overlap = tu > 0 ? both / tu : 0.0;
    r.g2c_overlap = td > 0 ? both / td : 0.0;
    // file lane vs the union of the two link lanes (merged into disjoint
    // intervals first: the link lanes overlap each other)
    std::sort(ssd.begin(), ssd.end());
    std::sort(link.begin(), link.end());
    std::vector<std::pair<std::uint64_t, std::uint64_t>> merged;
    for (const auto& iv : link) {
        if (!merged.empty() && iv.first <= merged.back().second)
            merged.back().second = std::max(merged.back().second, iv.second);
        else
            merged.push_back(iv);
    }
    double ssd_both = 0;
    for (std::size_t i = 0, j = 0; i < ssd.size() && j < merged.size();) {
        const std::uint64_t lo = std::max(ssd[i].first, merged[j].first);
        const std::uint64_t hi = std::min(ssd[i].second, merged[j].second);
        if (hi > lo) ssd_both += static_cast<double>(hi - lo);
        if (ssd[i].second < merged[j].second) ++i;
        else ++j;
    }
    const double ts = total(ssd);
    r.ssd_link_overlap = ts > 0 ? ssd_both / ts : 0.0;
    r.c2g_bytes = ub;
    r.g2c_bytes = db;
}

} // namespace offsim
