// ThreadSanitizer build only (scripts/tsan.sh): the host-side core and C ABI
// are built with -fsanitize=thread without the CUDA executor; offsim::execute
// is replaced by this stub so the C ABI links (offsim_execute then reports
// OFFSIM_ERR_INFEASIBLE, exactly as on a machine without a GPU).
#include "offsim/errors.hpp"
#include "offsim/exec.hpp"

namespace offsim {
ExecReport execute(const ModelConfig&, const HardwareConfig&, const SwapPlan&, ScheduleVariant,
                   const ExecOptions&, const std::vector<ChunkBuffers>*) {
    throw InfeasibleError("TSAN build: no CUDA executor");
}
} // namespace offsim
