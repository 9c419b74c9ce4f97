// Workload geometry, machine validation and presets — restates
// proj/src/workload.cpp, proj/src/hardware.cpp and proj/src/presets.cpp
// (same integer/double expressions, so every derived byte and FLOP count is
// identical; verified by tests/parity against the compiled reference).

#include "offsim/errors.hpp"
#include "offsim/hardware.hpp"
#include "offsim/presets.hpp"
#include "offsim/workload.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <sstream>

namespace offsim {

// ------------------------------------------------------------- workload

const char* to_string(LayerKind kind) {
    static constexpr std::array<const char*, 4> kNames = {"linear_qkv", "linear_htoh",
                                                          "linear_hto4h", "linear_4htoh"};
    const auto i = static_cast<std::size_t>(kind);
    return i < kNames.size() ? kNames[i] : "unknown";
}

void ModelConfig::validate() const {
    struct Rule {
        bool bad;
        const char* message;
    };
    const Rule rules[] = {
        {num_layers < 1, "model: num_layers must be >= 1"},
        {num_heads < 1, "model: num_heads must be >= 1"},
        {hidden_dim < 1, "model: hidden_dim must be >= 1"},
        {batch_size < 1, "model: batch_size must be >= 1"},
        {seq_len < 1, "model: seq_len must be >= 1"},
        {param_elem_bytes < 1, "model: param_elem_bytes must be >= 1"},
        {activation_elem_bytes < 1, "model: activation_elem_bytes must be >= 1"},
        {optimizer_state_multiplier <= 0.0, "model: optimizer_state_multiplier must be > 0"},
        {extra_flops_per_block < 0.0, "model: extra_flops_per_block must be >= 0"},
    };
    for (const Rule& r : rules)
        if (r.bad) throw ConfigError(r.message);
    // checked last: the modulo needs num_heads >= 1
    if (hidden_dim % num_heads != 0)
        throw ConfigError("model: hidden_dim must be divisible by num_heads");
}

std::uint64_t total_param_count(const ModelConfig& cfg) {
    return 12ull * cfg.num_layers * cfg.hidden_dim * cfg.hidden_dim;
}

namespace {

// Per-kind constants of a block's linear layers: output width (x h), weight
// count (x h^2), forward FLOPs (x b*s*h^2) and swap time (x t_s).
struct KindRow {
    LayerKind kind;
    std::uint64_t out_width;
    std::uint64_t weights;
    double flop_coeff;
    std::uint32_t swap_units;
};
constexpr std::array<KindRow, 4> kKinds = {{
    {LayerKind::linear_qkv, 3, 3, 6.0, 3},
    {LayerKind::linear_htoh, 1, 1, 2.0, 1},
    {LayerKind::linear_hto4h, 4, 4, 8.0, 4},
    {LayerKind::linear_4htoh, 1, 4, 8.0, 1},
}};

std::uint64_t block_weight_bytes(const ModelConfig& cfg) {
    return 12ull * cfg.hidden_dim * cfg.hidden_dim * cfg.param_elem_bytes;
}

std::uint64_t checkpoint_bytes(const ModelConfig& cfg) {
    return cfg.batch_size * cfg.seq_len * cfg.hidden_dim * cfg.activation_elem_bytes;
}

} // namespace

std::vector<LayerProfile> build_layer_profiles(const ModelConfig& cfg) {
    const std::uint64_t h = cfg.hidden_dim;
    const double bsh2 = static_cast<double>(cfg.batch_size) * static_cast<double>(cfg.seq_len) *
                        static_cast<double>(h) * static_cast<double>(h);
    const std::uint64_t token_bytes =
        cfg.batch_size * cfg.seq_len * static_cast<std::uint64_t>(cfg.activation_elem_bytes);
    std::vector<LayerProfile> profiles;
    profiles.reserve(4ull * cfg.num_layers);
    for (std::uint32_t blk = 0; blk < cfg.num_layers; ++blk) {
        for (const KindRow& row : kKinds) {
            LayerProfile lp;
            lp.block_index = blk;
            lp.kind = row.kind;
            lp.act_bytes = token_bytes * row.out_width * h;
            lp.param_bytes = row.weights * h * h * cfg.param_elem_bytes;
            lp.flops_fwd = row.flop_coeff * bsh2;
            lp.swap_time_units = row.swap_units;
            profiles.push_back(lp);
        }
    }
    return profiles;
}

FootprintReport footprint(const ModelConfig& cfg) {
    FootprintReport fp;
    fp.total_params = total_param_count(cfg);
    fp.fp16_param_bytes = fp.total_params * cfg.param_elem_bytes;
    fp.fp16_grad_bytes = fp.fp16_param_bytes;
    fp.optimizer_state_bytes = static_cast<std::uint64_t>(
        std::llround(static_cast<double>(fp.fp16_param_bytes) * cfg.optimizer_state_multiplier));
    fp.model_state_bytes = fp.fp16_param_bytes + fp.fp16_grad_bytes + fp.optimizer_state_bytes;
    fp.checkpoint_bytes_per_block = checkpoint_bytes(cfg);
    fp.total_checkpoint_bytes = fp.checkpoint_bytes_per_block * cfg.num_layers;
    return fp;
}

std::uint64_t total_intra_block_act_bytes(const ModelConfig& cfg) {
    return cfg.num_layers * cfg.batch_size * cfg.seq_len * 9ull * cfg.hidden_dim *
           cfg.activation_elem_bytes;
}

std::uint64_t gpu_working_set_bytes(const ModelConfig& cfg) {
    const std::uint64_t acts =
        cfg.batch_size * cfg.seq_len * 9ull * cfg.hidden_dim * cfg.activation_elem_bytes;
    const auto weights = static_cast<std::uint64_t>(
        std::llround(kResidentBlockMultiplier * static_cast<double>(block_weight_bytes(cfg))));
    return weights + acts + checkpoint_bytes(cfg);
}

// ------------------------------------------------------------- hardware

ValidationReport validate(const HardwareConfig& hw, const ModelConfig* paired_model) {
    ValidationReport report;
    const std::pair<double, const char*> must_be_positive[] = {
        {hw.bw_gpu, "bw_gpu"},
        {hw.bw_s2c, "bw_s2c"},
        {hw.bw_c2s, "bw_c2s"},
        {static_cast<double>(hw.gpu_mem), "gpu_mem"},
        {static_cast<double>(hw.cpu_mem), "cpu_mem"},
        {static_cast<double>(hw.ssd_capacity), "ssd_capacity"},
        {hw.gpu_tput, "gpu_tput"},
        {hw.cpu_opt_tput, "cpu_opt_tput"},
    };
    for (const auto& [value, field] : must_be_positive)
        if (!(value > 0.0)) report.errors.push_back(std::string(field) + " must be > 0");
    if (hw.n_ssd < 1) report.errors.push_back("n_ssd must be >= 1");
    const std::pair<double, const char*> non_negative[] = {
        {hw.gpu_price_dollars, "gpu_price_dollars"},
        {hw.ssd_price_dollars, "ssd_price_dollars"},
        {hw.server_price_dollars, "server_price_dollars"},
    };
    for (const auto& [value, field] : non_negative)
        if (value < 0.0) report.errors.push_back(std::string(field) + " must be >= 0");

    if (paired_model && report.ok()) {
        const std::uint64_t need = footprint(*paired_model).model_state_bytes;
        if (hw.ssd_capacity < need) {
            std::ostringstream os;
            os << "ssd_capacity " << hw.ssd_capacity << " is below the model-state bytes "
               << need << " of model '" << paired_model->name << "'";
            report.warnings.push_back(os.str());
        }
    }
    return report;
}

double aggregate_ssd_bw(const HardwareConfig& hw, SsdDirection dir) {
    return (dir == SsdDirection::s2c ? hw.bw_s2c : hw.bw_c2s) * static_cast<double>(hw.n_ssd);
}

// -------------------------------------------------------------- presets

namespace {

constexpr std::uint64_t kGB = 1000ull * 1000 * 1000;

struct ModelRow {
    const char* name;
    std::uint32_t layers, heads;
    std::uint64_t hidden;
};
constexpr std::array<ModelRow, 8> kModelRows = {{
    {"gpt3-13b", 40, 40, 5120},
    {"gpt3-33b", 60, 52, 6656},
    {"gpt3-65b", 80, 64, 8192},
    {"gpt3-135b", 88, 88, 11264},
    {"gpt3-175b", 96, 96, 12288},
    {"gpt3-276b", 112, 112, 14336},
    {"gpt3-412b", 128, 128, 16384},
    {"gpt3-805b", 160, 160, 20480},
}};

ModelConfig from_row(const ModelRow& r) {
    ModelConfig m;
    m.name = r.name;
    m.num_layers = r.layers;
    m.num_heads = r.heads;
    m.hidden_dim = r.hidden;
    m.batch_size = 1;
    m.seq_len = 1024;
    return m;
}

struct MachineRow {
    const char* name;
    std::uint64_t gpu_mem;
    double gpu_tput;
    double gpu_price;
};
constexpr std::array<MachineRow, 2> kMachineRows = {{
    {"a100-12ssd", 80 * kGB, 2.0e14, 14177.0},
    {"rtx4090-12ssd", 24 * kGB, 1.64e14, 1600.0},
}};

HardwareConfig from_row(const MachineRow& r) {
    // Shared chassis: PCIe Gen4 x16, 12 x 3.84 TB NVMe, 768 GB DRAM, CPU
    // optimizer at 1e9 params/s (calibration constants, proj/README.md).
    HardwareConfig hw;
    hw.name = r.name;
    hw.bw_gpu = 25e9;
    hw.bw_s2c = 6e9;
    hw.bw_c2s = 3e9;
    hw.n_ssd = 12;
    hw.gpu_mem = r.gpu_mem;
    hw.cpu_mem = 768 * kGB;
    hw.ssd_capacity = 12ull * 3840 * kGB;
    hw.gpu_tput = r.gpu_tput;
    hw.cpu_opt_tput = 1e9;
    hw.gpu_price_dollars = r.gpu_price;
    hw.ssd_price_dollars = 308.0;
    hw.server_price_dollars = 14098.0;
    return hw;
}

template <typename Rows>
std::vector<std::string> names_of(const Rows& rows) {
    std::vector<std::string> out;
    for (const auto& r : rows) out.emplace_back(r.name);
    return out;
}

} // namespace

const std::vector<std::string>& model_preset_names() {
    static const std::vector<std::string> names = names_of(kModelRows);
    return names;
}

ModelConfig model_preset(const std::string& name) {
    const auto it = std::find_if(kModelRows.begin(), kModelRows.end(),
                                 [&](const ModelRow& r) { return name == r.name; });
    if (it == kModelRows.end()) throw ConfigError("unknown model preset '" + name + "'");
    return from_row(*it);
}

const std::vector<std::string>& hardware_preset_names() {
    static const std::vector<std::string> names = names_of(kMachineRows);
    return names;
}

HardwareConfig hardware_preset(const std::string& name) {
    const auto it = std::find_if(kMachineRows.begin(), kMachineRows.end(),
                                 [&](const MachineRow& r) { return name == r.name; });
    if (it == kMachineRows.end()) throw ConfigError("unknown hardware preset '" + name + "'");
    return from_row(*it);
}

std::vector<ModelConfig> model_ladder() {
    std::vector<ModelConfig> ladder;
    for (const ModelRow& r : kModelRows) ladder.push_back(from_row(r));
    std::sort(ladder.begin(), ladder.end(), [](const ModelConfig& a, const ModelConfig& b) {
        return total_param_count(a) < total_param_count(b);
    });
    return ladder;
}

} // namespace offsim
