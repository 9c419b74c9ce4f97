// Closed-form cost model (paper Eqs. 2-11) and the swap planner (Eq. 12 +
// prefix search) — restates proj/src/cost_model.cpp and proj/src/planner.cpp.
// Floating-point expressions are evaluated in the same order as the
// reference so plans and predicted times agree to the last bit (pinned by
// tests/parity against the compiled reference over the acceptance matrix).

#include "offsim/cost_model.hpp"
#include "offsim/errors.hpp"
#include "offsim/planner.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <sstream>

namespace offsim {

const char* to_string(ForwardBottleneck b) {
    switch (b) {
    case ForwardBottleneck::gpu_compute: return "gpu_compute";
    case ForwardBottleneck::gpu_link: return "gpu_link";
    case ForwardBottleneck::ssd_link: return "ssd_link";
    }
    return "unknown";
}

const char* to_string(BackwardBottleneck b) {
    switch (b) {
    case BackwardBottleneck::gpu_compute: return "gpu_compute";
    case BackwardBottleneck::cpu_optimizer: return "cpu_optimizer";
    case BackwardBottleneck::gpu_link: return "gpu_link";
    case BackwardBottleneck::ssd_link: return "ssd_link";
    }
    return "unknown";
}

namespace {

struct SsdRates {
    double read, write;
};
SsdRates ssd_rates(const HardwareConfig& hw) {
    return {aggregate_ssd_bw(hw, SsdDirection::s2c), aggregate_ssd_bw(hw, SsdDirection::c2s)};
}

// Strictly-greater promotion over the terms in priority order: a later term
// is reported only when it beats every earlier one.
template <typename E, std::size_t N>
E dominant(const double (&t)[N], const E (&tags)[N]) {
    E tag = tags[0];
    double best = t[0];
    for (std::size_t i = 1; i < N; ++i) {
        if (t[i] > best) tag = tags[i];
        best = std::max(best, t[i]);
    }
    return tag;
}

} // namespace

ForwardTimes forward_time(const CostInputs& in, const HardwareConfig& hw) {
    const SsdRates ssd = ssd_rates(hw);
    const double w16 = 2.0 * in.total_params; // fp16 weight bytes streamed in
    ForwardTimes ft;
    ft.t_f_comp = in.fwd_flops / hw.gpu_tput;
    ft.t_f_gpu = std::max(w16 / hw.bw_gpu, in.d_f / hw.bw_gpu);
    ft.t_f_ssd = w16 / ssd.read + (in.checkpoints_on_ssd ? in.d_f / ssd.write : 0.0);
    ft.t_f = std::max({ft.t_f_comp, ft.t_f_gpu, ft.t_f_ssd});
    const double terms[3] = {ft.t_f_comp, ft.t_f_gpu, ft.t_f_ssd};
    const ForwardBottleneck tags[3] = {ForwardBottleneck::gpu_compute,
                                       ForwardBottleneck::gpu_link, ForwardBottleneck::ssd_link};
    ft.bottleneck = dominant(terms, tags);
    return ft;
}

BackwardOptimizerTimes backward_optimizer_time(const CostInputs& in, const HardwareConfig& hw) {
    const SsdRates ssd = ssd_rates(hw);
    const double p = in.total_params;
    const double w16 = 2.0 * p;
    BackwardOptimizerTimes bt;
    // backward = 2x forward FLOPs, plus recompute of unswapped layers
    bt.t_b_comp = 2.0 * in.fwd_flops / hw.gpu_tput + in.recompute_flops / hw.gpu_tput;
    // the optimizer lane: p params at cpu_opt_tput
    bt.t_o_comp = p / hw.cpu_opt_tput;
    bt.t_bo_gpu_g2c = w16 / hw.bw_gpu;
    bt.t_bo_gpu_c2g = (w16 + in.d_f) / hw.bw_gpu;
    bt.t_bo_gpu = std::max(w16 / hw.bw_gpu, (w16 + in.d_f) / hw.bw_gpu);
    // SSD: read 12p states + 2p weights (+ checkpoints), write 14p
    const double ckpt_ssd = in.checkpoints_on_ssd ? in.d_f : 0.0;
    bt.t_bo_ssd = (14.0 * p + ckpt_ssd) / ssd.read + 14.0 * p / ssd.write;
    bt.t_bo = std::max({bt.t_b_comp, bt.t_o_comp, bt.t_bo_gpu, bt.t_bo_ssd});
    const double terms[4] = {bt.t_b_comp, bt.t_o_comp, bt.t_bo_gpu, bt.t_bo_ssd};
    const BackwardBottleneck tags[4] = {BackwardBottleneck::gpu_compute,
                                        BackwardBottleneck::cpu_optimizer,
                                        BackwardBottleneck::gpu_link, BackwardBottleneck::ssd_link};
    bt.bottleneck = dominant(terms, tags);
    return bt;
}

CostBreakdown iteration_time(const CostInputs& in, const HardwareConfig& hw) {
    const ForwardTimes f = forward_time(in, hw);
    const BackwardOptimizerTimes b = backward_optimizer_time(in, hw);
    CostBreakdown c;
    c.t_f_comp = f.t_f_comp;
    c.t_f_gpu = f.t_f_gpu;
    c.t_f_ssd = f.t_f_ssd;
    c.t_f = f.t_f;
    c.t_b_comp = b.t_b_comp;
    c.t_o_comp = b.t_o_comp;
    c.t_bo_gpu = b.t_bo_gpu;
    c.t_bo_gpu_c2g = b.t_bo_gpu_c2g;
    c.t_bo_gpu_g2c = b.t_bo_gpu_g2c;
    c.t_bo_ssd = b.t_bo_ssd;
    c.t_bo = b.t_bo;
    c.t_iter = f.t_f + b.t_bo;
    c.d_f = in.d_f;
    c.bottleneck_f = f.bottleneck;
    c.bottleneck_bo = b.bottleneck;
    return c;
}

SwapBudget swap_budget(const CostInputs& at_start, const HardwareConfig& hw) {
    const BackwardOptimizerTimes b = backward_optimizer_time(at_start, hw);
    SwapBudget sb;
    sb.t_max_s = b.t_b_comp - std::max(b.t_bo_gpu, b.t_bo_ssd);
    if (sb.t_max_s <= 0.0) {
        sb.exhausted = true;
        sb.d_max_bytes = at_start.d_f;
        return sb;
    }
    const SsdRates ssd = ssd_rates(hw);
    sb.d_max_bytes = sb.t_max_s * std::min({hw.bw_gpu, ssd.write, ssd.read});
    return sb;
}

CostInputs make_cost_inputs(const ModelConfig& cfg,
                            const std::vector<std::uint32_t>& swapped_layers,
                            bool checkpoints_on_ssd) {
    const std::vector<LayerProfile> layers = build_layer_profiles(cfg);
    const FootprintReport fp = footprint(cfg);
    CostInputs ci;
    ci.total_params = static_cast<double>(fp.total_params);
    ci.checkpoints_on_ssd = checkpoints_on_ssd;
    double flops = 0.0;
    for (const LayerProfile& lp : layers) flops += lp.flops_fwd;
    flops += cfg.extra_flops_per_block * static_cast<double>(cfg.num_layers);
    ci.fwd_flops = flops;
    double saved = 0.0;
    std::uint64_t moved = 0;
    for (const std::uint32_t i : swapped_layers) {
        saved += layers.at(i).flops_fwd;
        moved += layers.at(i).act_bytes;
    }
    // attention extras are always recomputed; only linears can be swapped
    ci.recompute_flops = flops - saved;
    ci.d_f = static_cast<double>(fp.total_checkpoint_bytes + moved);
    return ci;
}

// ---------------------------------------------------------------- planner

double swap_benefit_factor(const LayerProfile& layer) {
    double coeff = 8.0; // linear_hto4h and linear_4htoh
    if (layer.kind == LayerKind::linear_qkv) coeff = 6.0;
    else if (layer.kind == LayerKind::linear_htoh) coeff = 2.0;
    const double unit_flops = layer.flops_fwd / coeff; // b*s*h^2
    const double per_swap_unit = layer.flops_fwd / static_cast<double>(layer.swap_time_units);
    return per_swap_unit / (2.0 * unit_flops);
}

PriorityQueues build_priority_queues(const std::vector<LayerProfile>& profiles) {
    PriorityQueues q;
    for (std::uint32_t i = 0; i < profiles.size(); ++i)
        (profiles[i].kind == LayerKind::linear_4htoh ? q.high : q.low).push_back(i);
    return q;
}

std::vector<std::uint32_t> PriorityQueues::order() const {
    std::vector<std::uint32_t> all;
    all.reserve(high.size() + low.size());
    all.insert(all.end(), high.begin(), high.end());
    all.insert(all.end(), low.begin(), low.end());
    return all;
}

SwapPlan plan_swaps(const ModelConfig& model, const HardwareConfig& hw,
                    const PlannerOptions& options) {
    model.validate();
    if (const ValidationReport r = validate(hw); !r.ok())
        throw ConfigError("hardware: " + r.errors.front());
    if (const std::uint64_t ws = gpu_working_set_bytes(model); ws > hw.gpu_mem) {
        std::ostringstream os;
        os << "model '" << model.name << "' cannot run at batch size " << model.batch_size
           << ": GPU working set " << ws << " exceeds gpu_mem " << hw.gpu_mem;
        throw InfeasibleError(os.str());
    }

    const std::vector<LayerProfile> layers = build_layer_profiles(model);
    const std::vector<std::uint32_t> order = build_priority_queues(layers).order();
    const FootprintReport fp = footprint(model);
    const std::uint64_t intra = total_intra_block_act_bytes(model);

    const CostInputs base = make_cost_inputs(model, {}, options.checkpoints_on_ssd);
    const SwapBudget budget = swap_budget(base, hw);
    const BackwardOptimizerTimes b0 = backward_optimizer_time(base, hw);
    const double ssd_read = aggregate_ssd_bw(hw, SsdDirection::s2c);
    const double w16 = 2.0 * base.total_params;

    const bool automatic = options.mode == PlannerOptions::Mode::automatic;
    double cap = std::numeric_limits<double>::infinity();
    switch (options.mode) {
    case PlannerOptions::Mode::automatic: break;
    case PlannerOptions::Mode::fixed_d_f:
        cap = std::max(options.fixed_d_f_bytes, base.d_f);
        break;
    case PlannerOptions::Mode::fixed_coefficient:
        if (options.fixed_coefficient < 0.0 || options.fixed_coefficient > 1.0)
            throw ConfigError("planner: fixed coefficient must be in [0, 1]");
        cap = base.d_f + options.fixed_coefficient * static_cast<double>(intra) + 0.5;
        break;
    }

    // Running terms of the backward stage as the swapped prefix grows by one
    // layer per iteration; the forward stage is re-evaluated each time.
    double comp = b0.t_b_comp;
    double link = b0.t_bo_gpu;
    double ssd = b0.t_bo_ssd;
    double d_f = base.d_f;
    std::size_t chosen = 0;
    double best = std::numeric_limits<double>::infinity();
    for (std::size_t prefix = 0; prefix <= order.size(); ++prefix) {
        if (prefix > 0) {
            const LayerProfile& added = layers[order[prefix - 1]];
            comp -= added.flops_fwd / hw.gpu_tput;
            d_f += static_cast<double>(added.act_bytes);
            link = std::max(w16 / hw.bw_gpu, (w16 + d_f) / hw.bw_gpu);
            if (options.checkpoints_on_ssd) ssd += static_cast<double>(added.act_bytes) / ssd_read;
        }
        if (automatic && prefix > 0 && d_f > budget.d_max_bytes) break;
        if (d_f > cap) break;
        CostInputs here = base;
        here.d_f = d_f;
        const double t_iter = forward_time(here, hw).t_f + std::max({comp, b0.t_o_comp, link, ssd});
        if (!automatic) {
            chosen = prefix; // fixed modes: longest prefix under the cap
        } else if (t_iter < best) {
            best = t_iter;
            chosen = prefix; // ties keep the smaller prefix
        }
    }

    SwapPlan plan;
    plan.d_start_bytes = fp.total_checkpoint_bytes;
    plan.t_max_s = budget.t_max_s;
    plan.d_max_bytes = budget.d_max_bytes;
    plan.checkpoints_on_ssd = options.checkpoints_on_ssd;
    plan.swapped_layers.assign(order.begin(), order.begin() + static_cast<std::ptrdiff_t>(chosen));
    std::uint64_t moved = 0;
    for (const std::uint32_t i : plan.swapped_layers) moved += layers[i].act_bytes;
    plan.d_f_bytes = fp.total_checkpoint_bytes + moved;
    plan.swap_coefficient =
        intra == 0 ? 0.0 : static_cast<double>(moved) / static_cast<double>(intra);
    plan.predicted =
        iteration_time(make_cost_inputs(model, plan.swapped_layers, options.checkpoints_on_ssd), hw);
    return plan;
}

} // namespace offsim
