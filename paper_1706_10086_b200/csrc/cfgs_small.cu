// cfgs_small.cu -- TMA configurations with 128x64 / 64x128 / 64x64 / 32x64 CTA tiles (mid-size and small problems;
// 64x64 with E=16 is the paper's P100 optimum, 16x16 threads x T=4, Tab. 4).
#include "registry.cuh"

namespace dg {

static const CfgEntry k_table[] = {
    DG_TMA(128, 64, 16, 64, 32, 4),
    DG_TMA(128, 64, 16, 32, 32, 6),
    DG_TMA(128, 64, 16, 32, 16, 6),
    DG_TMA(64, 128, 16, 32, 64, 4),
    DG_TMA_XP(64, 128, 16, 32, 64, 4),
    DG_TMA_XP(64, 64, 16, 32, 16, 6),
    DG_TMA(64, 128, 16, 32, 32, 6),
    DG_TMA(64, 128, 16, 16, 32, 6),
    DG_TMA(64, 64, 16, 64, 32, 6),
    DG_TMA(64, 64, 16, 32, 32, 6),
    DG_TMA(64, 64, 16, 32, 16, 6),
    DG_TMA(64, 64, 16, 16, 32, 6),
    DG_TMA_SPLIT(64, 64, 16, 32, 16, 6),
    DG_TMA_SPLIT(128, 64, 16, 32, 16, 6),
    DG_TMA_SPLIT(64, 128, 16, 32, 64, 4),
    DG_TMA_SPLIT(128, 128, 16, 32, 32, 4),
    DG_SK(64, 64, 16, 32, 16, 6),
    DG_SK(128, 64, 16, 32, 16, 6),
    DG_HYB(64, 64, 16, 32, 16, 6),
    DG_TMA(64, 64, 32, 16, 32, 3),
    DG_TMA_SPLIT(64, 64, 32, 32, 16, 3),
    DG_HYB(64, 64, 32, 32, 16, 3),
    // round 2: BK = 32 stream-K (small shapes whose operands stay in L2) and E = 32 tiles
    DG_SK(64, 64, 32, 32, 16, 3),
    DG_SK(64, 64, 32, 16, 32, 3),
    DG_SK(128, 64, 32, 32, 32, 3),
    DG_TMA_SPLIT(128, 64, 32, 32, 32, 3),
    // one 16-warp CTA per SM (E = 16): no co-resident CTA to share the DMMA pipe unevenly
    DG_SK(128, 64, 32, 32, 16, 4),
    DG_SK(64, 128, 32, 16, 32, 4),
    DG_TMA_SPLIT(128, 64, 32, 32, 16, 4),
    // cluster split-K: the slices of a tile reduce through distributed shared memory
    DG_CSK(64, 64, 32, 32, 16, 3),
    DG_CSK(64, 64, 16, 32, 16, 6),
    DG_CSK(128, 64, 32, 32, 32, 3),
    // round 2: 32x64 / 64x32 / 32x32 tiles with E = 8 (16x16 warp tiles, 8 warps): twice the
    // tiles of 64x64 at the same shape, so small problems fill the SMs with fewer (or no) split-K
    // slices and no reduction (512^3: 128 tiles, one pass; DESIGN.md §6 small shapes, round 2)
    DG_TMA_SPLIT(32, 64, 32, 16, 16, 3),
    DG_TMA_SPLIT(32, 64, 32, 16, 16, 4),
    DG_TMA_SPLIT(32, 64, 64, 16, 16, 3),
    DG_TMA_SPLIT(64, 32, 32, 16, 16, 4),
    DG_TMA_SPLIT(32, 32, 32, 16, 16, 4),
    DG_TMA(32, 64, 32, 16, 16, 3),
    DG_HYB(32, 64, 32, 16, 16, 3),
    DG_SK(32, 64, 32, 16, 16, 3),
    // three CTAs per SM (64 registers; tuner-only: with three slots per SM the block scheduler packs
    // a grid that fits onto fewer SMs, DESIGN.md §6 small shapes (10))
    DG_TMA_SPLIT_MB(32, 64, 32, 16, 16, 3, 3),
    DG_TMA_MB(32, 64, 32, 16, 16, 3, 3),
    DG_TMA_SPLIT_MB(32, 64, 32, 16, 16, 2, 3),
};

const CfgEntry *cfg_table_small(int *n) {
    *n = (int)(sizeof(k_table) / sizeof(k_table[0]));
    return k_table;
}

}  // namespace dg
