// Schedule builder — restates proj/src/task_graph.cpp:122-506.
//
// Emits the iteration's task DAG in the reference's exact task order (task
// ids, names, dependency lists and memory effects are part of the executor
// contract and of the bit-exact parity suite):
//   forward   per linear: p_s2c -> p_c2g -> compute, swapped act_g2c[->c2s],
//             per block ckpt_g2c[->c2s]                       (:254-322)
//   backward  blocks in reverse: param fetch, checkpoint / activation
//             restore, recompute, 4 backward computes, grad_g2c
//             [+ grad_c2s when not overlapped]                 (:327-451)
//   optimizer groups in reverse: [grad_s2c,] state_s2c, update, state_c2s,
//             param_c2s; read gate depth 2 (delayed write-back) (:453-503)
// The B200 executor (exec.cpp) runs the optimizer and activation-swap tasks
// of this graph for real.

#include "offsim/errors.hpp"
#include "offsim/sim.hpp"

#include <algorithm>
#include <cmath>
#include <sstream>

namespace offsim {

const char* to_string(ResourceId id) {
    switch (id) {
    case ResourceId::gpu_compute: return "gpu_compute";
    case ResourceId::cpu_compute: return "cpu_compute";
    case ResourceId::link_c2g: return "link_c2g";
    case ResourceId::link_g2c: return "link_g2c";
    case ResourceId::link_ssd: return "link_ssd";
    case ResourceId::mem_gpu: return "mem_gpu";
    case ResourceId::mem_cpu: return "mem_cpu";
    }
    return "unknown";
}

const char* to_string(TaskKind kind) {
    switch (kind) {
    case TaskKind::compute: return "compute";
    case TaskKind::transfer: return "transfer";
    case TaskKind::optimizer_update: return "optimizer_update";
    }
    return "unknown";
}

const char* to_string(TransferDir dir) {
    switch (dir) {
    case TransferDir::none: return "none";
    case TransferDir::s2c: return "s2c";
    case TransferDir::c2s: return "c2s";
    case TransferDir::c2g: return "c2g";
    case TransferDir::g2c: return "g2c";
    }
    return "unknown";
}

const char* to_string(Payload p) {
    switch (p) {
    case Payload::none: return "none";
    case Payload::params: return "params";
    case Payload::grads: return "grads";
    case Payload::opt_states: return "opt_states";
    case Payload::activations: return "activations";
    }
    return "unknown";
}

const char* to_string(ScheduleVariant v) {
    switch (v) {
    case ScheduleVariant::serial: return "serial";
    case ScheduleVariant::pipelined: return "pipelined";
    case ScheduleVariant::overlapped: return "overlapped";
    }
    return "unknown";
}

ScheduleVariant schedule_variant_from_string(const std::string& s) {
    for (ScheduleVariant v :
         {ScheduleVariant::serial, ScheduleVariant::pipelined, ScheduleVariant::overlapped})
        if (s == to_string(v)) return v;
    throw ConfigError("unknown schedule variant '" + s + "'");
}

namespace {

constexpr std::uint32_t kAbsent = 0xffffffffu;
using Ids = std::vector<std::uint32_t>;

MemEffect on_gpu(std::int64_t bytes, bool at_start) {
    return MemEffect{ResourceId::mem_gpu, bytes, at_start};
}
MemEffect on_cpu(std::int64_t bytes, bool at_start) {
    return MemEffect{ResourceId::mem_cpu, bytes, at_start};
}

// Window of `unit`-sized items that fit `budget`, clamped to [lo, hi].
std::uint32_t fit_window(std::uint64_t budget, std::uint64_t unit, std::uint32_t lo,
                         std::uint32_t hi) {
    const std::uint64_t n = unit == 0 ? hi : budget / unit;
    return static_cast<std::uint32_t>(std::clamp<std::uint64_t>(n, lo, hi));
}

class Builder {
public:
    Builder(const ModelConfig& model, const HardwareConfig& hw, const SwapPlan& plan,
            ScheduleVariant variant, const BuildOptions& opts)
        : model_(model), hw_(hw), plan_(plan), variant_(variant), opts_(opts) {}

    TaskGraph build();

private:
    // Appends one task; deps are cleaned (absent ids dropped, sorted,
    // de-duplicated) and, for the serial variant, chained to the previous
    // task so nothing overlaps.
    std::uint32_t emit(std::string name, TaskKind kind, ResourceId lane, TransferDir dir,
                       Payload payload, double work, Ids deps, std::vector<MemEffect> fx) {
        Task t;
        t.id = static_cast<std::uint32_t>(g_.tasks.size());
        if (serial_ && t.id > 0) deps.push_back(t.id - 1);
        deps.erase(std::remove(deps.begin(), deps.end(), kAbsent), deps.end());
        std::sort(deps.begin(), deps.end());
        deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
        t.name = std::move(name);
        t.kind = kind;
        t.resource = lane;
        t.dir = dir;
        t.payload = payload;
        t.work = work;
        t.deps = std::move(deps);
        t.mem_effects = std::move(fx);
        g_.tasks.push_back(std::move(t));
        return g_.tasks.back().id;
    }

    std::string layer_tag(std::uint32_t i) const {
        std::ostringstream os;
        os << "b" << layers_[i].block_index << " " << to_string(layers_[i].kind);
        return os.str();
    }
    static std::string block_tag(char prefix, std::uint32_t k) {
        std::ostringstream os;
        os << prefix << k;
        return os.str();
    }
    std::int64_t act(std::uint32_t i) const { return static_cast<std::int64_t>(layers_[i].act_bytes); }
    std::int64_t wts(std::uint32_t i) const { return static_cast<std::int64_t>(layers_[i].param_bytes); }

    void size_windows();
    void forward();
    void backward();
    void optimizer();

    const ModelConfig& model_;
    const HardwareConfig& hw_;
    const SwapPlan& plan_;
    ScheduleVariant variant_;
    BuildOptions opts_;
    TaskGraph g_;

    std::vector<LayerProfile> layers_;
    FootprintReport fp_;
    std::vector<bool> swapped_;
    std::uint32_t blocks_ = 0, linears_ = 0;
    bool serial_ = false, overlapped_ = false, ckpt_ssd_ = false;
    std::uint64_t fifo_ = 0, block_w_bytes_ = 0, block_opt_bytes_ = 0;
    double block_params_ = 0.0;
    std::int64_t ckpt_ = 0;
    std::uint32_t w_prefetch_ = 1, w_offload_ = 1, w_bwd_ = 1, w_stage_ = 1;

    // Producer ids shared between phases.
    Ids fwd_comp_, ckpt_out_, ckpt_g2c_, act_out_, act_g2c_;
    Ids bwd_done_, grad_g2c_, grad_c2s_;
    std::uint32_t fwd_last_ = kAbsent;
};

void Builder::size_windows() {
    const std::uint64_t ws = gpu_working_set_bytes(model_);
    if (ws > hw_.gpu_mem) {
        std::ostringstream os;
        os << "GPU working set " << ws << " exceeds gpu_mem " << hw_.gpu_mem;
        throw InfeasibleError(os.str());
    }
    fifo_ = hw_.gpu_mem - ws;

    // The prefetcher must be able to hold its largest single unit.
    std::uint64_t largest = fp_.checkpoint_bytes_per_block;
    std::uint32_t largest_at = 0;
    std::uint64_t largest_weights = 0;
    for (std::uint32_t i = 0; i < linears_; ++i) {
        largest_weights = std::max(largest_weights, layers_[i].param_bytes);
        const std::uint64_t unit =
            swapped_[i] ? std::max(layers_[i].param_bytes, layers_[i].act_bytes)
                        : layers_[i].param_bytes;
        if (unit > largest) {
            largest = unit;
            largest_at = i;
        }
    }
    if (fifo_ < largest) {
        std::ostringstream os;
        os << "GPU FIFO capacity " << fifo_ << " cannot hold the prefetch unit of layer "
           << layer_tag(largest_at) << " (" << largest << " bytes)";
        throw InfeasibleError(os.str());
    }

    block_w_bytes_ = 12ull * model_.hidden_dim * model_.hidden_dim * model_.param_elem_bytes;
    block_opt_bytes_ = static_cast<std::uint64_t>(std::llround(
        static_cast<double>(block_w_bytes_) * model_.optimizer_state_multiplier));
    block_params_ = 12.0 * static_cast<double>(model_.hidden_dim) *
                    static_cast<double>(model_.hidden_dim);

    std::uint64_t restore_max = 0;
    for (std::uint32_t k = 0; k < blocks_; ++k) {
        std::uint64_t r = fp_.checkpoint_bytes_per_block;
        for (std::uint32_t j = 0; j < 4; ++j)
            if (swapped_[4 * k + j]) r += layers_[4 * k + j].act_bytes;
        restore_max = std::max(restore_max, r);
    }
    w_prefetch_ = fit_window(fifo_ * 2 / 5, largest_weights, 1, linears_);
    w_offload_ = fit_window(fifo_ / 2, restore_max, 1, blocks_);
    w_bwd_ = fit_window(fifo_ / 2, block_w_bytes_ + restore_max, 1,
                        std::min<std::uint32_t>(blocks_, 4));

    const double ssd_read = aggregate_ssd_bw(hw_, SsdDirection::s2c);
    const double ratio = hw_.bw_gpu / ssd_read;
    const std::uint64_t cpu_queue =
        std::min(static_cast<std::uint64_t>(static_cast<double>(fifo_) * ratio), hw_.cpu_mem / 4);
    w_stage_ = fit_window(cpu_queue, largest_weights, 1, linears_);

    const std::uint64_t staging = 4 * (block_w_bytes_ * 2 + block_opt_bytes_) + cpu_queue;
    if (serial_ && plan_.d_f_bytes + staging > hw_.cpu_mem) {
        std::ostringstream os;
        os << "checkpoints (" << plan_.d_f_bytes << " bytes) plus staging (" << staging
           << ") exceed cpu_mem " << hw_.cpu_mem << " with CPU-resident placement";
        throw InfeasibleError(os.str());
    }
}

void Builder::forward() {
    fwd_comp_.assign(linears_, kAbsent);
    ckpt_out_.assign(blocks_, kAbsent);
    ckpt_g2c_.assign(blocks_, kAbsent);
    act_out_.assign(linears_, kAbsent);
    act_g2c_.assign(linears_, kAbsent);

    for (std::uint32_t i = 0; i < linears_; ++i) {
        const std::uint32_t blk = i / 4, pos = i % 4;
        const std::string tag = layer_tag(i);
        const double wbytes = static_cast<double>(layers_[i].param_bytes);

        Ids read_deps;
        if (!serial_ && i >= w_prefetch_ + w_stage_)
            read_deps.push_back(fwd_comp_[i - w_prefetch_ - w_stage_]);
        const std::uint32_t s2c =
            emit("fwd p_s2c " + tag, TaskKind::transfer, ResourceId::link_ssd, TransferDir::s2c,
                 Payload::params, wbytes, std::move(read_deps), {on_cpu(wts(i), false)});

        Ids up_deps{s2c};
        if (!serial_ && i >= w_prefetch_) up_deps.push_back(fwd_comp_[i - w_prefetch_]);
        const std::uint32_t c2g =
            emit("fwd p_c2g " + tag, TaskKind::transfer, ResourceId::link_c2g, TransferDir::c2g,
                 Payload::params, wbytes, std::move(up_deps),
                 {on_gpu(wts(i), true), on_cpu(-wts(i), false)});

        Ids comp_deps{c2g};
        if (i > 0) comp_deps.push_back(fwd_comp_[i - 1]);
        if (!serial_ && pos == 0 && blk >= w_offload_) comp_deps.push_back(ckpt_g2c_[blk - w_offload_]);
        std::vector<MemEffect> fx{on_gpu(-wts(i), false)};
        if (swapped_[i]) fx.push_back(on_gpu(act(i), false));
        double flops = layers_[i].flops_fwd;
        if (pos == 3) {
            fx.push_back(on_gpu(ckpt_, false));
            flops += model_.extra_flops_per_block;
        }
        fwd_comp_[i] = emit("fwd compute " + tag, TaskKind::compute, ResourceId::gpu_compute,
                            TransferDir::none, Payload::none, flops, std::move(comp_deps),
                            std::move(fx));

        if (swapped_[i]) {
            const double abytes = static_cast<double>(layers_[i].act_bytes);
            act_g2c_[i] = emit("fwd act_g2c " + tag, TaskKind::transfer, ResourceId::link_g2c,
                               TransferDir::g2c, Payload::activations, abytes, {fwd_comp_[i]},
                               {on_cpu(act(i), true), on_gpu(-act(i), false)});
            act_out_[i] = act_g2c_[i];
            if (ckpt_ssd_)
                act_out_[i] = emit("fwd act_c2s " + tag, TaskKind::transfer, ResourceId::link_ssd,
                                   TransferDir::c2s, Payload::activations, abytes, {act_g2c_[i]},
                                   {on_cpu(-act(i), false)});
        }
        if (pos == 3) {
            const std::string btag = block_tag('b', blk);
            const double cbytes = static_cast<double>(fp_.checkpoint_bytes_per_block);
            ckpt_g2c_[blk] = emit("fwd ckpt_g2c " + btag, TaskKind::transfer, ResourceId::link_g2c,
                                  TransferDir::g2c, Payload::activations, cbytes, {fwd_comp_[i]},
                                  {on_cpu(ckpt_, true), on_gpu(-ckpt_, false)});
            ckpt_out_[blk] = ckpt_g2c_[blk];
            if (ckpt_ssd_)
                ckpt_out_[blk] = emit("fwd ckpt_c2s " + btag, TaskKind::transfer,
                                      ResourceId::link_ssd, TransferDir::c2s, Payload::activations,
                                      cbytes, {ckpt_g2c_[blk]}, {on_cpu(-ckpt_, false)});
        }
    }
    fwd_last_ = fwd_comp_[linears_ - 1];
}

void Builder::backward() {
    bwd_done_.assign(blocks_, kAbsent);
    grad_g2c_.assign(blocks_, kAbsent);
    grad_c2s_.assign(blocks_, kAbsent);
    const std::int64_t grad_bytes = static_cast<std::int64_t>(block_w_bytes_);
    const double cbytes = static_cast<double>(fp_.checkpoint_bytes_per_block);

    for (std::uint32_t m = 0; m < blocks_; ++m) {
        const std::uint32_t kb = blocks_ - 1 - m;
        // Restores of this block wait until the block w_bwd_ ahead (in
        // processing order) has finished its backward computes.
        const std::uint32_t gate = (!serial_ && m >= w_bwd_) ? bwd_done_[kb + w_bwd_] : fwd_last_;
        const Ids gated = serial_ ? Ids{} : Ids{gate};

        Ids w_up(4, kAbsent);
        for (std::uint32_t j = 0; j < 4; ++j) {
            const std::uint32_t i = 4 * kb + j;
            const std::string tag = layer_tag(i);
            const double wbytes = static_cast<double>(layers_[i].param_bytes);
            const std::uint32_t rd =
                emit("bwd p_s2c " + tag, TaskKind::transfer, ResourceId::link_ssd,
                     TransferDir::s2c, Payload::params, wbytes, gated, {on_cpu(wts(i), false)});
            w_up[j] = emit("bwd p_c2g " + tag, TaskKind::transfer, ResourceId::link_c2g,
                           TransferDir::c2g, Payload::params, wbytes, {rd},
                           {on_gpu(wts(i), true), on_cpu(-wts(i), false)});
        }

        const std::string btag = block_tag('b', kb);
        std::uint32_t ck_src = ckpt_out_[kb];
        if (ckpt_ssd_)
            ck_src = emit("bwd ckpt_s2c " + btag, TaskKind::transfer, ResourceId::link_ssd,
                          TransferDir::s2c, Payload::activations, cbytes,
                          serial_ ? Ids{ckpt_out_[kb]} : Ids{ckpt_out_[kb], gate},
                          {on_cpu(ckpt_, false)});
        const std::uint32_t ck_up =
            emit("bwd ckpt_c2g " + btag, TaskKind::transfer, ResourceId::link_c2g,
                 TransferDir::c2g, Payload::activations, cbytes,
                 (ckpt_ssd_ || serial_) ? Ids{ck_src} : Ids{ck_src, gate},
                 {on_gpu(ckpt_, true), on_cpu(-ckpt_, false)});

        Ids act_up(4, kAbsent);
        for (std::uint32_t j = 0; j < 4; ++j) {
            const std::uint32_t i = 4 * kb + j;
            if (!swapped_[i]) continue;
            const std::string tag = layer_tag(i);
            const double abytes = static_cast<double>(layers_[i].act_bytes);
            std::uint32_t src = act_out_[i];
            if (ckpt_ssd_)
                src = emit("bwd act_s2c " + tag, TaskKind::transfer, ResourceId::link_ssd,
                           TransferDir::s2c, Payload::activations, abytes,
                           serial_ ? Ids{act_out_[i]} : Ids{act_out_[i], gate},
                           {on_cpu(act(i), false)});
            act_up[j] = emit("bwd act_c2g " + tag, TaskKind::transfer, ResourceId::link_c2g,
                             TransferDir::c2g, Payload::activations, abytes,
                             (ckpt_ssd_ || serial_) ? Ids{src} : Ids{src, gate},
                             {on_gpu(act(i), true), on_cpu(-act(i), false)});
        }

        // Recompute the discarded activations in forward order; producer of
        // layer j's output is either its restore or its recompute.
        Ids produced(4, kAbsent);
        std::uint32_t prev = ck_up;
        for (std::uint32_t j = 0; j < 4; ++j) {
            const std::uint32_t i = 4 * kb + j;
            if (swapped_[i]) {
                produced[j] = prev = act_up[j];
                continue;
            }
            double flops = layers_[i].flops_fwd;
            if (j == 3) flops += model_.extra_flops_per_block;
            produced[j] = prev = emit("bwd recompute " + layer_tag(i), TaskKind::compute,
                                      ResourceId::gpu_compute, TransferDir::none, Payload::none,
                                      flops, {w_up[j], prev}, {});
        }

        // Backward computes, last layer first.
        std::uint32_t dgrad = (kb == blocks_ - 1) ? fwd_last_ : bwd_done_[kb + 1];
        for (std::int32_t j = 3; j >= 0; --j) {
            const auto ju = static_cast<std::uint32_t>(j);
            const std::uint32_t i = 4 * kb + ju;
            Ids deps{w_up[ju], dgrad, j == 0 ? ck_up : produced[ju - 1]};
            if (swapped_[i]) deps.push_back(act_up[ju]);
            std::vector<MemEffect> fx{on_gpu(-wts(i), false)};
            if (swapped_[i]) fx.push_back(on_gpu(-act(i), false));
            double flops = 2.0 * layers_[i].flops_fwd;
            if (j == 3) flops += 2.0 * model_.extra_flops_per_block;
            if (j == 0) {
                fx.push_back(on_gpu(-ckpt_, false));
                fx.push_back(on_gpu(grad_bytes, false));
            }
            dgrad = emit("bwd compute " + layer_tag(i), TaskKind::compute, ResourceId::gpu_compute,
                         TransferDir::none, Payload::none, flops, std::move(deps), std::move(fx));
        }
        bwd_done_[kb] = dgrad;

        grad_g2c_[kb] = emit("bwd grad_g2c " + btag, TaskKind::transfer, ResourceId::link_g2c,
                             TransferDir::g2c, Payload::grads, static_cast<double>(block_w_bytes_),
                             {bwd_done_[kb]}, {on_cpu(grad_bytes, true), on_gpu(-grad_bytes, false)});
        if (!overlapped_)
            grad_c2s_[kb] = emit("bwd grad_c2s " + btag, TaskKind::transfer, ResourceId::link_ssd,
                                 TransferDir::c2s, Payload::grads,
                                 static_cast<double>(block_w_bytes_), {grad_g2c_[kb]},
                                 {on_cpu(-grad_bytes, false)});
    }
}

void Builder::optimizer() {
    const std::int64_t states = static_cast<std::int64_t>(block_opt_bytes_);
    const std::int64_t grad_bytes = static_cast<std::int64_t>(block_w_bytes_);
    const double wbytes = static_cast<double>(block_w_bytes_);
    Ids update(blocks_, kAbsent);
    const std::uint32_t all_backward = overlapped_ ? kAbsent : grad_c2s_[0];

    for (std::uint32_t m = 0; m < blocks_; ++m) {
        const std::uint32_t kb = blocks_ - 1 - m;
        const std::string gtag = block_tag('g', kb);
        // Read gate: two groups ahead of the update pipeline.
        Ids gate;
        if (overlapped_)
            gate.push_back(m >= 2 ? grad_g2c_[blocks_ - 1 - (m - 2)] : fwd_last_);
        else if (!serial_)
            gate.push_back(all_backward);
        if (!serial_ && m >= 2) gate.push_back(update[blocks_ - 1 - (m - 2)]);

        std::uint32_t grad_src = kAbsent;
        if (!overlapped_) {
            Ids deps = gate;
            deps.push_back(grad_c2s_[kb]);
            grad_src = emit("opt grad_s2c " + gtag, TaskKind::transfer, ResourceId::link_ssd,
                            TransferDir::s2c, Payload::grads, wbytes, std::move(deps),
                            {on_cpu(grad_bytes, false)});
        }
        const std::uint32_t rd =
            emit("opt state_s2c " + gtag, TaskKind::transfer, ResourceId::link_ssd,
                 TransferDir::s2c, Payload::opt_states, static_cast<double>(block_opt_bytes_),
                 Ids(gate), {on_cpu(states, false)});
        // The gradient buffer turns into the updated low-precision weights
        // of equal size: net zero on CPU memory.
        update[kb] = emit("opt update " + gtag, TaskKind::optimizer_update,
                          ResourceId::cpu_compute, TransferDir::none, Payload::none, block_params_,
                          {rd, overlapped_ ? grad_g2c_[kb] : grad_src},
                          {on_cpu(-grad_bytes, false), on_cpu(grad_bytes, false)});
        emit("opt state_c2s " + gtag, TaskKind::transfer, ResourceId::link_ssd, TransferDir::c2s,
             Payload::opt_states, static_cast<double>(block_opt_bytes_), {update[kb]},
             {on_cpu(-states, false)});
        emit("opt param_c2s " + gtag, TaskKind::transfer, ResourceId::link_ssd, TransferDir::c2s,
             Payload::params, wbytes, {update[kb]}, {on_cpu(-grad_bytes, false)});
    }
}

TaskGraph Builder::build() {
    model_.validate();
    if (const ValidationReport r = validate(hw_); !r.ok())
        throw ConfigError("hardware: " + r.errors.front());

    layers_ = build_layer_profiles(model_);
    fp_ = footprint(model_);
    blocks_ = model_.num_layers;
    linears_ = static_cast<std::uint32_t>(layers_.size());
    swapped_.assign(linears_, false);
    for (const std::uint32_t i : plan_.swapped_layers) swapped_.at(i) = true;
    serial_ = variant_ == ScheduleVariant::serial;
    overlapped_ = variant_ == ScheduleVariant::overlapped;
    // serial keeps checkpoints in CPU memory; the others follow the plan
    ckpt_ssd_ = !serial_ && plan_.checkpoints_on_ssd;
    ckpt_ = static_cast<std::int64_t>(fp_.checkpoint_bytes_per_block);

    size_windows();

    TraceHeader& h = g_.header;
    h.variant = variant_;
    h.model_name = model_.name;
    h.hardware_name = hw_.name;
    h.checkpoint_location = ckpt_ssd_ ? "ssd" : "cpu";
    h.fp16_param_bytes = fp_.fp16_param_bytes;
    h.gpu_fifo_bytes = fifo_;
    h.prefetch_window_layers = w_prefetch_;
    h.offload_window_blocks = w_offload_;
    h.cpu_stage_window_layers = w_stage_;
    h.forward_only = opts_.forward_only;
    // Two block-weight slots of the working set are modelled by task
    // effects (active weights, gradients); the rest is a static reservation.
    g_.initial_mem[ResourceId::mem_gpu] =
        static_cast<std::int64_t>(gpu_working_set_bytes(model_) - 2 * block_w_bytes_);
    g_.initial_mem[ResourceId::mem_cpu] = 0;

    forward();
    if (opts_.forward_only) return std::move(g_);
    backward();
    optimizer();
    return std::move(g_);
}

} // namespace

TaskGraph build_schedule(const ModelConfig& model, const HardwareConfig& hw,
                         const SwapPlan& plan, ScheduleVariant variant,
                         const BuildOptions& options) {
    return Builder(model, hw, plan, variant, options).build();
}

} // namespace offsim
