// offsim public C++ API — all declarations in one header.
//
// Declaration-compatible with the reference's per-topic headers
// (proj/include/offsim/{errors,workload,hardware,presets,cost_model,
// planner,sim,scenario,capacity,runner}.hpp): every type, field, enumerator
// and function signature a reference caller uses exists here unchanged, so
// the reference's own test suites compile against it. The per-topic headers
// in this directory are kept as one-line forwarders for source
// compatibility. The B200 execution layer is declared in offsim/exec.hpp.
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace offsim {

// ======================================================================
// Errors — offsim error taxonomy — declaration-compatible with the reference
// (proj/include/offsim/errors.hpp:9-30). Status codes of the C ABI and the
// CLI exit codes derive from the dynamic type: ConfigError -> 2,
// InfeasibleError -> 3, InvariantError -> 4.
// ======================================================================

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Input that is malformed or self-inconsistent (scenario document, model or
// hardware field, unknown preset / variant / key).
struct ConfigError : Error {
    using Error::Error;
};

// A well-formed scenario that cannot be executed on the machine it names:
// GPU working set or FIFO too small, CPU-resident checkpoints too large, and
// on the B200 executor also a device / pinned-host allocation that fails.
struct InfeasibleError : Error {
    using Error::Error;
};

// A schedule or trace broke one of its invariants (deadlock, pool overflow,
// dependency or exclusivity violation in an executed trace).
struct InvariantError : Error {
    using Error::Error;
};

// ======================================================================
// Workload geometry — Transformer workload geometry (declaration-compatible
// with the reference proj/include/offsim/workload.hpp). One transformer
// block is one optimizer chunk of 12h^2 parameters: [qkv 3h^2 | htoh h^2 |
// hto4h 4h^2 | 4htoh 4h^2].
// ======================================================================

// The block's four linear layers, in forward execution order.
enum class LayerKind : std::uint8_t {
    linear_qkv,   // h -> 3h
    linear_htoh,  // h -> h
    linear_hto4h, // h -> 4h
    linear_4htoh, // 4h -> h
};

const char* to_string(LayerKind kind);

struct ModelConfig {
    std::string name;
    std::uint32_t num_layers = 1; // transformer blocks = optimizer chunks
    std::uint32_t num_heads = 1;
    std::uint64_t hidden_dim = 1;
    std::uint64_t batch_size = 1;
    std::uint64_t seq_len = 1;

    // Bytes per low-precision weight; optimizer state is this many times the
    // weight bytes (fp32 master + m + v = 12 B per 2-B weight).
    std::uint32_t param_elem_bytes = 2;
    double optimizer_state_multiplier = 6.0;

    // Activation bytes per element (1 => a (b, s, h) tensor is b*s*h bytes).
    std::uint32_t activation_elem_bytes = 1;

    // Additional forward FLOPs per block (attention scores), 0 by default.
    double extra_flops_per_block = 0.0;

    void validate() const; // throws ConfigError
};

struct LayerProfile {
    std::uint32_t block_index = 0;
    LayerKind kind = LayerKind::linear_qkv;
    std::uint64_t act_bytes = 0;
    std::uint64_t param_bytes = 0;
    double flops_fwd = 0.0;
    std::uint32_t swap_time_units = 1;
};

struct FootprintReport {
    std::uint64_t total_params = 0;
    std::uint64_t fp16_param_bytes = 0;
    std::uint64_t fp16_grad_bytes = 0;
    std::uint64_t optimizer_state_bytes = 0;
    std::uint64_t model_state_bytes = 0;
    std::uint64_t checkpoint_bytes_per_block = 0;
    std::uint64_t total_checkpoint_bytes = 0;
};

// p = 12 * layers * h^2 (linears only).
std::uint64_t total_param_count(const ModelConfig& cfg);

// 4 * layers profiles: block-major, forward order inside a block.
std::vector<LayerProfile> build_layer_profiles(const ModelConfig& cfg);

FootprintReport footprint(const ModelConfig& cfg);

// b * s * 9h * act_elem per block, summed over blocks.
std::uint64_t total_intra_block_act_bytes(const ModelConfig& cfg);

// Resident GPU bytes while one block runs: kResidentBlockMultiplier block
// weight buffers + one block's activations + one checkpoint.
std::uint64_t gpu_working_set_bytes(const ModelConfig& cfg);

inline constexpr double kResidentBlockMultiplier = 4.0;

// ======================================================================
// Machine — Machine description (declaration-compatible with the reference
// proj/include/offsim/hardware.hpp). Rates are sustained figures: the DES
// prices tasks with them and the B200 executor is calibrated against them.
// ======================================================================

struct HardwareConfig {
    std::string name;
    double bw_gpu = 0.0; // host link, bytes/s in each direction (duplex)
    double bw_s2c = 0.0; // per-SSD read bytes/s
    double bw_c2s = 0.0; // per-SSD write bytes/s
    std::uint32_t n_ssd = 1;
    std::uint64_t gpu_mem = 0;
    std::uint64_t cpu_mem = 0;
    std::uint64_t ssd_capacity = 0; // whole array
    double gpu_tput = 0.0;          // FLOP/s
    double cpu_opt_tput = 0.0;      // optimizer params/s (the optimizer lane)

    double gpu_price_dollars = 0.0;
    double ssd_price_dollars = 0.0;    // each
    double server_price_dollars = 0.0; // chassis only
};

enum class SsdDirection : std::uint8_t { s2c, c2s };

struct ValidationReport {
    std::vector<std::string> errors;
    std::vector<std::string> warnings;
    bool ok() const { return errors.empty(); }
};

ValidationReport validate(const HardwareConfig& hw, const ModelConfig* paired_model = nullptr);

// Per-device rate x device count.
double aggregate_ssd_bw(const HardwareConfig& hw, SsdDirection dir);

// ======================================================================
// Presets — Named models and machines (declaration-compatible with the
// reference proj/include/offsim/presets.hpp).
// ======================================================================

// GPT-3 family shapes at seq_len 1024, batch 1.
const std::vector<std::string>& model_preset_names();
ModelConfig model_preset(const std::string& name); // ConfigError if unknown

// Commodity PCIe Gen4 server with a 12-SSD array, A100 or RTX 4090.
const std::vector<std::string>& hardware_preset_names();
HardwareConfig hardware_preset(const std::string& name); // ConfigError if unknown

// Model presets ordered by parameter count, ascending.
std::vector<ModelConfig> model_ladder();

// ======================================================================
// Closed-form cost model — Closed-form iteration model, paper Eqs. 2-11
// (declaration-compatible with the reference
// proj/include/offsim/cost_model.hpp). Each stage time is the maximum over
// its resources; the backward stage overlaps the optimizer.
// ======================================================================

enum class ForwardBottleneck : std::uint8_t { gpu_compute, gpu_link, ssd_link };
enum class BackwardBottleneck : std::uint8_t { gpu_compute, cpu_optimizer, gpu_link, ssd_link };

const char* to_string(ForwardBottleneck b);
const char* to_string(BackwardBottleneck b);

struct CostInputs {
    double total_params = 0.0;
    double fwd_flops = 0.0;
    double recompute_flops = 0.0;
    double d_f = 0.0; // checkpoint + swapped activation bytes, one way
    bool checkpoints_on_ssd = true;
};

struct ForwardTimes {
    double t_f = 0.0;
    double t_f_comp = 0.0;
    double t_f_gpu = 0.0;
    double t_f_ssd = 0.0;
    ForwardBottleneck bottleneck = ForwardBottleneck::gpu_compute;
};

struct BackwardOptimizerTimes {
    double t_bo = 0.0;
    double t_b_comp = 0.0;
    double t_o_comp = 0.0;
    double t_bo_gpu = 0.0;
    double t_bo_ssd = 0.0;
    double t_bo_gpu_c2g = 0.0;
    double t_bo_gpu_g2c = 0.0;
    BackwardBottleneck bottleneck = BackwardBottleneck::gpu_compute;
};

struct CostBreakdown {
    double t_f_comp = 0.0;
    double t_f_gpu = 0.0;
    double t_f_ssd = 0.0;
    double t_f = 0.0;
    double t_b_comp = 0.0;
    double t_o_comp = 0.0;
    double t_bo_gpu = 0.0;
    double t_bo_gpu_c2g = 0.0;
    double t_bo_gpu_g2c = 0.0;
    double t_bo_ssd = 0.0;
    double t_bo = 0.0;
    double t_iter = 0.0;
    double d_f = 0.0;
    ForwardBottleneck bottleneck_f = ForwardBottleneck::gpu_compute;
    BackwardBottleneck bottleneck_bo = BackwardBottleneck::gpu_compute;
};

ForwardTimes forward_time(const CostInputs& in, const HardwareConfig& hw);
BackwardOptimizerTimes backward_optimizer_time(const CostInputs& in, const HardwareConfig& hw);
CostBreakdown iteration_time(const CostInputs& in, const HardwareConfig& hw);

struct SwapBudget {
    double t_max_s = 0.0;
    double d_max_bytes = 0.0;
    bool exhausted = false;
};

// `at_start` is the one-checkpoint-per-block volume (d_f = D_start).
SwapBudget swap_budget(const CostInputs& at_start, const HardwareConfig& hw);

// `swapped_layers` indexes build_layer_profiles(cfg).
CostInputs make_cost_inputs(const ModelConfig& cfg,
                            const std::vector<std::uint32_t>& swapped_layers,
                            bool checkpoints_on_ssd = true);

// ======================================================================
// Swap planner — Activation swap planner, paper Eq. 12 + prefix search
// (declaration- compatible with the reference
// proj/include/offsim/planner.hpp). Its decisions must match the reference
// bit for bit; the B200 executor only carries them out.
// ======================================================================

struct SwapPlan {
    std::uint64_t d_start_bytes = 0;
    std::uint64_t d_f_bytes = 0;
    double d_max_bytes = 0.0;
    double t_max_s = 0.0;
    std::vector<std::uint32_t> swapped_layers; // prefix of the priority order
    double swap_coefficient = 0.0;             // swapped / all intra-block act bytes
    bool checkpoints_on_ssd = true;
    CostBreakdown predicted;
};

double swap_benefit_factor(const LayerProfile& layer);

struct PriorityQueues {
    std::vector<std::uint32_t> high; // every linear_4htoh, block order
    std::vector<std::uint32_t> low;  // the rest, block order
    std::vector<std::uint32_t> order() const;
};
PriorityQueues build_priority_queues(const std::vector<LayerProfile>& profiles);

struct PlannerOptions {
    enum class Mode : std::uint8_t { automatic, fixed_d_f, fixed_coefficient };
    Mode mode = Mode::automatic;
    double fixed_d_f_bytes = 0.0;
    double fixed_coefficient = 0.0;
    bool checkpoints_on_ssd = true;
};

SwapPlan plan_swaps(const ModelConfig& model, const HardwareConfig& hw,
                    const PlannerOptions& options = {});

// ======================================================================
// Task graph, traces, DES, validation — Task graph, traces, the discrete-
// event simulator and the trace validator (declaration-compatible with the
// reference proj/include/offsim/sim.hpp). The same TaskGraph / SimTrace
// types are the contract of the B200 executor (offsim/exec.hpp): it fills
// TraceEvent times from CUDA events instead of integer-ns arithmetic, and
// check_trace_invariants validates both.
// ======================================================================

// Serial lanes (first five) and capacity pools (last two).
enum class ResourceId : std::uint8_t {
    gpu_compute,
    cpu_compute,
    link_c2g,
    link_g2c,
    link_ssd,
    mem_gpu,
    mem_cpu,
};
const char* to_string(ResourceId id);

enum class TaskKind : std::uint8_t { compute, transfer, optimizer_update };
const char* to_string(TaskKind kind);

enum class TransferDir : std::uint8_t { none, s2c, c2s, c2g, g2c };
const char* to_string(TransferDir dir);

enum class Payload : std::uint8_t { none, params, grads, opt_states, activations };
const char* to_string(Payload p);

struct MemEffect {
    ResourceId mem = ResourceId::mem_gpu;
    std::int64_t delta_bytes = 0;
    bool at_start = false;
};

struct Task {
    std::uint32_t id = 0;
    std::string name;
    TaskKind kind = TaskKind::compute;
    ResourceId resource = ResourceId::gpu_compute;
    TransferDir dir = TransferDir::none;
    Payload payload = Payload::none;
    double work = 0.0; // bytes, FLOPs or params
    std::vector<std::uint32_t> deps;
    std::vector<MemEffect> mem_effects;
};

enum class ScheduleVariant : std::uint8_t { serial, pipelined, overlapped };
const char* to_string(ScheduleVariant v);
ScheduleVariant schedule_variant_from_string(const std::string& s); // ConfigError

struct TraceHeader {
    ScheduleVariant variant = ScheduleVariant::overlapped;
    std::string model_name;
    std::string hardware_name;
    std::string checkpoint_location; // "cpu" | "ssd"
    std::uint64_t fp16_param_bytes = 0;
    std::uint64_t gpu_fifo_bytes = 0;
    std::uint32_t prefetch_window_layers = 0;
    std::uint32_t offload_window_blocks = 0;
    std::uint32_t cpu_stage_window_layers = 0;
    bool forward_only = false;
};

struct TaskGraph {
    TraceHeader header;
    std::vector<Task> tasks;
    std::map<ResourceId, std::int64_t> initial_mem;
};

struct BuildOptions {
    bool forward_only = false;
};

// Expands (model, plan, variant) into the iteration's task DAG (forward,
// backward in reverse block order, one optimizer group per block).
TaskGraph build_schedule(const ModelConfig& model, const HardwareConfig& hw,
                         const SwapPlan& plan, ScheduleVariant variant,
                         const BuildOptions& options = {});

struct TraceEvent {
    std::uint32_t task_id = 0;
    ResourceId resource = ResourceId::gpu_compute;
    TransferDir dir = TransferDir::none;
    Payload payload = Payload::none;
    double work = 0.0;
    std::uint64_t start_ns = 0;
    std::uint64_t end_ns = 0;
};

struct SimTrace {
    TraceHeader header;
    std::vector<TraceEvent> events; // completion order
    std::uint64_t makespan_ns = 0;
    std::map<ResourceId, std::int64_t> peak_mem;
    std::map<ResourceId, std::uint64_t> busy_ns;
    double makespan_s() const { return static_cast<double>(makespan_ns) * 1e-9; }
};

std::uint64_t task_duration_ns(const Task& task, const HardwareConfig& hw);

SimTrace simulate(const TaskGraph& graph, const HardwareConfig& hw);

std::uint64_t serial_duration_sum_ns(const TaskGraph& graph, const HardwareConfig& hw);

std::uint64_t roofline_lower_bound_ns(const TaskGraph& graph, const HardwareConfig& hw);

struct InvariantReport {
    struct Entry {
        std::string name;
        bool pass = false;
        std::string detail;
    };
    std::vector<Entry> entries;
    bool all_pass = true;
};

InvariantReport check_trace_invariants(const TaskGraph& graph, const SimTrace& trace,
                                       const HardwareConfig& hw);

std::string to_chrome_trace_json(const TaskGraph& graph, const SimTrace& trace);

// ======================================================================
// Scenario documents — Scenario documents, schema v1 (declaration-compatible
// with the reference proj/include/offsim/scenario.hpp).
// ======================================================================

inline constexpr int kScenarioSchemaVersion = 1;

struct Scenario {
    int schema_version = kScenarioSchemaVersion;
    ModelConfig model;
    HardwareConfig hardware;
    ScheduleVariant variant = ScheduleVariant::overlapped;
    PlannerOptions::Mode planner_mode = PlannerOptions::Mode::automatic;
    double planner_value = 0.0;
    std::int64_t seed = 0;
};

Scenario load_scenario(const std::string& json_text);   // ConfigError
std::string scenario_to_json(const Scenario& s);        // round-trips

const std::vector<std::string>& scenario_preset_names();
Scenario scenario_preset(const std::string& name); // ConfigError

// ======================================================================
// Capacity and cost-effectiveness — Capacity and cost-effectiveness analysis
// (declaration-compatible with the reference
// proj/include/offsim/capacity.hpp). Not on the optimizer hot path; kept so
// the C ABI (offsim_capacity, offsim_sweep) is complete.
// ======================================================================

enum class PolicyId : std::uint8_t { zero_infinity, two_level };
const char* to_string(PolicyId id);
PolicyId policy_from_string(const std::string& s);

inline constexpr double kZeroInfinityCpuBytesPerParam = 5.0;
inline constexpr double kCpuStagingGroups = 4.0;

enum class CapacityBottleneck : std::uint8_t { none, ssd, cpu_mem, gpu_mem };
const char* to_string(CapacityBottleneck b);

struct PlacementBudget {
    std::uint64_t ssd_bytes = 0;
    std::uint64_t cpu_bytes = 0;
    std::uint64_t gpu_bytes = 0;
    bool checkpoints_on_ssd = false;
};
PlacementBudget placement_budget(PolicyId policy, const ModelConfig& model,
                                 const HardwareConfig& hw);

struct Feasibility {
    bool ok = false;
    CapacityBottleneck bottleneck = CapacityBottleneck::none;
    std::string detail;
};
Feasibility feasible(PolicyId policy, const ModelConfig& model, const HardwareConfig& hw);

struct MaxTrainable {
    bool found = false;
    ModelConfig model;
    CapacityBottleneck limit = CapacityBottleneck::none;
};
MaxTrainable max_trainable(PolicyId policy, const HardwareConfig& hw,
                           const std::vector<ModelConfig>& candidates);

struct PriceTable {
    double gpu = 0.0;
    double ssd = 0.0;
    double server = 0.0;
};
PriceTable price_table(const HardwareConfig& hw);

enum class PriceScope : std::uint8_t { gpu_ssd, whole_server };

double tokens_per_second(const ModelConfig& model, double t_iter_s);

double cost_effectiveness(double t_iter_s, const ModelConfig& model, const PriceTable& prices,
                          PriceScope scope, std::uint32_t n_ssd);

// ======================================================================
// Orchestration and reports — Orchestration (declaration-compatible with the
// reference proj/include/offsim/runner.hpp): placement, planning, schedule,
// DES, validation, and the JSON/CSV reports behind the C ABI.
// ======================================================================

// All-or-nothing checkpoint placement: CPU when the largest possible swap
// volume fits next to the optimizer staging groups, otherwise SSD.
bool checkpoints_fit_cpu(const ModelConfig& model, const HardwareConfig& hw);

SwapPlan plan_for_scenario(const Scenario& s);

struct RunOutputs {
    SwapPlan plan;
    TaskGraph graph;
    SimTrace trace;
    InvariantReport invariants;
};

RunOutputs run_scenario(const Scenario& s);

std::string plan_report_json(const Scenario& s);
std::string simulate_summary_json(const Scenario& s, std::string* trace_json_out);
std::string sweep_csv(const Scenario& base, const std::string& axis,
                      const std::vector<double>& values, int workers);
std::string capacity_csv(const Scenario& base, const std::vector<double>& cpu_mem_gb);
std::string validate_report_json(const Scenario& s);

} // namespace offsim
