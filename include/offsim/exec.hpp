// B200 executor — the real counterpart of simulate().
//
//   SimTrace simulate(const TaskGraph&, const HardwareConfig&)   (reference)
//   ExecReport execute(model, hw, plan, variant, ExecOptions)     (this)
//
// The reference prices a CPU optimizer and an SSD array; on B200 the Adam
// step runs on the GPU (fused kernel), so the executor first rewrites the
// reference task graph with a *tier map* (map_graph_for_b200) and then runs
// every task of the mapped graph on real engines:
//
//   reference task                      B200 operation (lane in the trace)
//   opt update gK   (cpu_compute)       fused AdamW kernel, optimizer stream
//                                       (cpu_compute lane = "optimizer")
//   + inserted opt state_h2d gK         H2D of [master|m|v] (link_c2g)
//   + inserted opt state_d2h gK         D2H of the updated states (link_g2c)
//   + inserted opt param_d2h gK         D2H of the bf16 params (link_g2c)
//   bwd grad_g2c / grad_c2s / grad_s2c  no bytes: grads stay in HBM (A5)
//   *_s2c / *_c2s on link_ssd           tier "file": pread/pwrite (O_DIRECT)
//                                       of real files; tier "host": no bytes
//                                       (the pinned host DRAM *is* the tier)
//   p_c2g / ckpt_c2g / act_c2g          H2D copy engine (link_c2g)
//   act_g2c / ckpt_g2c                  D2H copy engine (link_g2c)
//   fwd/bwd compute, recompute          synthetic compute: a timed kernel of
//                                       work / compute_rate seconds
//
// Every inserted task carries explicit dependencies, so the mapped graph is
// an ordinary TaskGraph: the executed trace is validated by the UNCHANGED
// check_trace_invariants against a HardwareConfig of measured B200 rates,
// and the report lists reference-graph bytes and physically moved bytes
// separately. Issue order on each engine follows simulate() of the mapped
// graph, so real execution replays the planned schedule.
#pragma once

#include "offsim/hardware.hpp"
#include "offsim/planner.hpp"
#include "offsim/sim.hpp"
#include "offsim/workload.hpp"

#include <cstdint>
#include <map>
#include <string>
#include <vector>

namespace offsim {

enum class StateTier : std::uint8_t { host, file };
const char* to_string(StateTier t);

struct AdamHyper {
    float lr = 1e-4f;
    float beta1 = 0.9f;
    float beta2 = 0.95f;
    float eps = 1e-8f;
    float weight_decay = 0.1f;
    std::uint64_t step = 10;
    bool adamw_mode = true;
    bool bias_correction = true;
    float grad_scale = 1.0f;
};

struct ExecOptions {
    int device = 0;
    StateTier tier = StateTier::host;
    std::string file_dir = "/tmp/offsim_b200";
    std::vector<std::string> file_dirs; // >1: tier files striped RAID-0 over these (one per SSD)
    bool direct_io = true;          // O_DIRECT for the file tier
    bool fixed_buffers = true;      // register the staging rings with io_uring (READ/WRITE_FIXED)
    std::uint32_t io_depth = 32;    // io_uring requests in flight PER tier device (file_dirs entry)
    // Before calibration and the timed iteration, bring the file lane to the
    // state every iteration after the first finds it: each activation /
    // checkpoint / gradient file extent written once and each host buffer a
    // file read lands in DMA-written once. Cold, the first write to a new
    // extent and the first device DMA into a host region run ~1.6x slower on
    // the leases' virtio disk (profiles/r02aq_file_rw_*.txt), so a single
    // cold iteration would measure first-touch costs, not the file lane.
    bool warm_files = true;
    double compute_rate = 0.0;      // FLOP/s of synthetic compute (0: hw.gpu_tput)
    // fwd/bwd compute tasks: "spin" = timed kernel of work / compute_rate
    // (no SM/HBM contention); "gemm" = the layer's real bf16 GEMMs through
    // cuBLAS (fwd: one b*s x out x in GEMM; bwd: dgrad + wgrad), so the
    // optimizer overlaps real tensor-core work (rate measured, not assumed);
    // "gemm_dataflow" = "gemm" with each layer's wgrad (X^T dY) written into
    // its block's gradient buffer, so the fused optimizer consumes the
    // gradients the backward produced (checked against an independent
    // computation of their norm).
    std::string compute_mode = "spin";
    std::uint32_t state_slots = 3;  // device staging slots for optimizer groups
    AdamHyper adam;
    std::uint64_t seed = 0;         // synthetic states / grads / activations
    bool verify_swaps = true;       // checksum every restored activation
    // Activation-swap sweep mode (BASELINE config 5): execute only the
    // activation / checkpoint transfers (swap_subgraph) of blocks < max_blocks
    // (0 = all blocks).
    bool swap_only = false;
    std::uint32_t max_blocks = 0;
    // File tier with bounded pinned staging (the SSD tier proper): 0 keeps a
    // host copy of every chunk; N > 0 stages optimizer states, params and
    // weights through N-slot pinned rings (and activations too when the
    // plan places them on SSD), so host memory no longer scales with the
    // model. Ring reuse is expressed as graph edges (add_host_ring_edges).
    std::uint32_t host_ring = 0;
    // host_ring "auto": per-ring depths from the reference schedule's own
    // windows (host_ring_depths) instead of one uniform N.
    bool host_ring_auto = false;
    // Report an FNV-1a checksum of every chunk's final [master|m|v].
    bool checksum_states = false;
    // Optimizer groups g0..g(R-1) whose states stay resident in HBM (see
    // map_graph_for_b200); 0xffffffff = all groups ("all"); kResidentAuto =
    // as many as the HBM left after the executor's own buffers holds ("auto").
    std::uint32_t resident_groups = 0;
    // "graph": the iteration is captured once into one CUDA graph and
    // launched as a unit (no host issue latency between tasks; falls back to
    // "stream" if the capture is refused); "stream": tasks issued one by one
    // on the lane streams in planned start order
    std::string launch = "graph";
};

inline constexpr std::uint32_t kResidentAuto = 0xfffffffeu;

// Caller-provided optimizer states for chunk (block) k: pinned host
// [master | m | v] (12n B) and the bf16 param output (2n B). When absent the
// executor allocates and seeds them itself.
struct ChunkBuffers {
    void* host_states = nullptr;
    void* host_params = nullptr;
    const void* device_grads = nullptr; // bf16 [n]; synthetic when null
};

// Graph rewrite only (no device needed): inserted hop tasks, zeroed byte
// counts for transfers that do not physically happen on B200 under `tier`.
// The m-th optimizer group (processing order) stages its states in device
// slot m % state_slots; the slot-reuse edge is part of the mapped graph.
// resident_groups: optimizer groups g0 .. g(R-1) keep master / m / v in HBM
// for the whole run (B200's HBM holds what the schedule leaves free): their
// state_h2d / state_d2h (and, file tier, state_s2c / state_c2s) move 0 B and
// their 12N B are booked in the GPU pool from the start (initial_mem).
TaskGraph map_graph_for_b200(const TaskGraph& graph, StateTier tier,
                             std::uint32_t state_slots = 3, std::uint32_t resident_groups = 0);

// Slot-reuse edges of the bounded host staging rings (file tier): the n-th
// use of a ring waits for the last task of use n - slots. Uses are, in task
// id order: optimizer groups (state_s2c .. state_c2s), param write-backs
// (param_d2h .. param_c2s), weight fetches (p_s2c .. p_c2g) and, when
// checkpoints live on SSD, activation transfers (g2c .. c2s, s2c .. c2g).
void add_host_ring_edges(TaskGraph& mapped, std::uint32_t slots);

// Slot counts of the four staging rings (0 = that ring is unused).
struct RingDepths {
    std::uint32_t states = 0;  // optimizer groups [master|m|v]
    std::uint32_t params = 0;  // bf16 param write-backs
    std::uint32_t weights = 0; // layer weight fetches (p_s2c .. p_c2g)
    std::uint32_t acts = 0;    // activations / checkpoints, placement = ssd
};
void add_host_ring_edges(TaskGraph& mapped, const RingDepths& depths);

// Ring depths of `mapped` under `opts` (all zero unless tier = file and
// host_ring > 0 or host_ring_auto). Uniform: host_ring slots per ring. Auto,
// from the windows build_schedule sized (task_graph.cpp:145-224, recorded in
// the graph header): weights = the CPU stage window in blocks
// (ceil(cpu_stage_window_layers / 4)); acts = the offload window
// (offload_window_blocks) times the activation units per block; states and
// params = the device staging slots (the optimizer's depth-2 read gate plus
// one write-back in flight). Every depth is at least 2 and at most the
// number of uses of its ring.
RingDepths host_ring_depths(const TaskGraph& mapped, const ExecOptions& opts);

// The activation-swap path of a (mapped) graph: every task with payload
// activations whose block index is < max_blocks (0 = all), dependencies
// restricted to the kept tasks (the swap-out -> [file] -> restore chains).
TaskGraph swap_subgraph(const TaskGraph& graph, std::uint32_t max_blocks);

// HardwareConfig describing the B200 box for the mapped graph's DES order
// and invariant checks (measured rates override the preset's).
struct MeasuredRates {
    double h2d_bps = 0.0;
    double d2h_bps = 0.0;
    double file_read_bps = 0.0;
    double file_write_bps = 0.0;
    double optimizer_params_per_s = 0.0;
    double compute_flops = 0.0;
    double compute_headroom = 1.0;  // compute_flops = measured x this (gemm mode)
    // the graph's own compute tasks replayed back to back (per-kernel
    // overhead and small-GEMM efficiency included)
    double compute_effective_flops = 0.0;
    std::uint64_t gpu_mem = 0;
    std::uint64_t cpu_mem = 0;
    // Delivered link rates when this graph's own host<->device copies run
    // back to back on both lanes at once (duplex, real copy sizes): what an
    // overlapped schedule actually gets from PCIe, vs the simplex burst
    // rates above.
    // the graph's own copies of one direction while the other direction is
    // continuously busy (duplex contention)
    double h2d_effective_bps = 0.0;
    double d2h_effective_bps = 0.0;
    // the same copies replayed one direction at a time (per-copy overhead,
    // no duplex contention)
    double h2d_simplex_effective_bps = 0.0;
    double d2h_simplex_effective_bps = 0.0;
    // share of each link lane's planned busy time during which the other
    // direction is also busy (link_overlap on the planned trace); the
    // effective rate of a lane blends its simplex and duplex replays by it
    double c2g_overlap = 1.0;
    double g2c_overlap = 1.0;
    double c2g_bytes = 0.0, g2c_bytes = 0.0;  // planned bytes per lane
    // file tier: this graph's own file-lane operations replayed in task order
    double file_read_effective_bps = 0.0;
    double file_write_effective_bps = 0.0;
    // ... and replayed again while both copy engines stream pinned host
    // memory (GPU DMA contends with the file device for host memory)
    double file_read_loaded_bps = 0.0;
    double file_write_loaded_bps = 0.0;
    // share of the file lane's planned busy time during which a link lane
    // is busy (link_overlap on the planned trace)
    double ssd_link_overlap = 0.0;
};
// Upper-bound rates (burst x 1.05): the issue order and the unchanged
// roofline-lower-bound invariant on the real trace.
HardwareConfig b200_hardware(const HardwareConfig& planned_on, const MeasuredRates& r);
// Effective rates (duplex link, measured kernel / compute, no headroom): the
// reference's DES on these predicts the executed makespan (SURVEY §8f
// rank 3: analytic vs executed).
HardwareConfig b200_hardware_effective(const HardwareConfig& planned_on, const MeasuredRates& r);
// Fills r.c2g_overlap / g2c_overlap / c2g_bytes / g2c_bytes from a trace of
// `graph` (the DES on the burst rates: where the two copy directions overlap).
void link_overlap(const TaskGraph& graph, const SimTrace& trace, MeasuredRates& r);

// The reference's analytic cost model (cost_model.cpp:26-90: t_iter =
// t_f + t_bo, each phase the max over its lanes of work / rate) applied to
// the B200-mapped graph: per phase (forward = "fwd ..." tasks; backward +
// optimizer = "bwd ..." / "opt ..." tasks), the busiest lane's summed task
// durations on `hw`. Same structure as iteration_time, but over the bytes
// the B200 execution actually moves (state hops on the host link, resident
// groups moving nothing), so it is comparable with an executed makespan.
struct AnalyticTimes {
    double t_f = 0.0;   // forward phase
    double t_bo = 0.0;  // backward + optimizer phase
    double t_iter = 0.0;
    std::string bottleneck_f, bottleneck_bo;  // lane names
};
AnalyticTimes analytic_iteration(const TaskGraph& mapped, const HardwareConfig& hw);

struct ExecReport {
    TaskGraph graph;        // the mapped graph that ran
    SimTrace trace;         // real timings (CUDA events), same type as simulate()
    SimTrace planned;       // simulate() of the mapped graph on `hw_exec`
    SimTrace predicted;     // simulate() of the mapped graph on `hw_predicted`
    InvariantReport invariants;
    HardwareConfig hw_exec;
    HardwareConfig hw_predicted;
    HardwareConfig hw_scenario;  // the scenario's own hardware (e.g. a persisted measured preset)
    SimTrace scenario_predicted; // simulate() of the mapped graph on hw_scenario
    MeasuredRates rates;         // the in-run calibration behind hw_exec / hw_predicted
    std::map<std::string, double> reference_bytes; // "<lane>/<payload>" of the input graph
    std::map<std::string, double> physical_bytes;  // "h2d|d2h|file_read|file_write/<payload>"
    double grad_sq_sum = 0.0;
    // compute_mode "gemm_dataflow": the grad sum of squares the backward's
    // wgrad GEMMs must hand the optimizer (computed independently before the
    // run); -1 otherwise
    double expected_grad_sq_sum = -1.0;
    int nonfinite = 0;
    std::uint64_t swap_checks = 0;     // restored buffers verified
    std::uint64_t swap_mismatches = 0; // must be 0
    std::uint32_t kernel_launches = 0;
    std::string io_engine; // "io_uring" | "pread/pwrite" (file tier)
    std::uint32_t file_devices = 0;        // tier files striped over this many directories
    std::uint64_t io_registered_bytes = 0; // staging rings registered with io_uring
    std::uint64_t io_fixed_requests = 0;   // file requests issued as READ/WRITE_FIXED
    std::uint64_t io_plain_requests = 0;   // ... and as plain READ/WRITE
    double file_warmup_s = 0.0;            // warm_files: untimed setup IO before calibration
    std::uint64_t pinned_host_bytes = 0;  // host staging the run allocated
    RingDepths host_ring;                 // staging ring depths (file tier)
    std::uint64_t state_checksum = 0;     // checksum_states
    std::uint32_t resident_groups = 0;    // optimizer groups kept in HBM
    std::string launch_mode;              // "graph" | "stream" (what actually ran)
};

ExecReport execute(const ModelConfig& model, const HardwareConfig& hw, const SwapPlan& plan,
                   ScheduleVariant variant, const ExecOptions& options,
                   const std::vector<ChunkBuffers>* chunks = nullptr);

std::string exec_summary_json(const ExecReport& r);

} // namespace offsim
