/* Compiled by tests/test_c_header.py: the INTEGRATION.md §4 caller, as plain
 * C11 against include/fuyou/fy_adam.h + include/offsim/offsim_c.h, linked
 * against the product library (no GPU needed to build). */
#include "offsim/offsim_c.h"
#include <stdint.h>
#include <stdio.h>
#include "fuyou/fy_adam.h"

int run(int local_rank, uint32_t W, uint32_t r, const void* id, uint32_t L, uint64_t* elems,
        void** my_states, void** grad_event, const fy_adam_hparams* hp, void* stream) {
    fy_shard_config cfg = {.device = local_rank, .world = W, .rank = r,
                           .gather = FY_GATHER_PEER, .nccl_id = id, .tier = FY_TIER_DEVICE,
                           .chunk_count = L, .chunk_elems = elems,
                           .grad_dtype = FY_BF16, .param_dtype = FY_BF16};
    fy_shard* sh;
    if (fy_shard_create(&cfg, &sh) != FY_OK) return 1;
    fy_shard_io io[64];
    for (uint32_t c = 0; c < L; ++c) {
        fy_shard_slice s;
        fy_shard_slice_info(sh, c, &s);
        io[c].states = my_states[c];
        io[c].grad = (uint16_t*)s.params + r * s.stride;
        io[c].h_param = 0;
        io[c].grad_ready = grad_event[c];
    }
    fy_shard_step(sh, io, hp, 1, stream);
    double sq; int bad;
    fy_shard_wait(sh, &sq, &bad);
    printf("%g %d\n", sq, bad);
    fy_shard_destroy(sh);
    return 0;
}
int main(void) { return 0; }
