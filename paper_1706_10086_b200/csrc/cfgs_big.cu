// cfgs_big.cu -- TMA configurations with 128x128 / 256x64 CTA tiles (large problems).
// E=16 at these tile sizes needs 32 warps -> 64 registers/thread -> spills; not instantiated.
#include "registry.cuh"

namespace dg {

static const CfgEntry k_table[] = {
    DG_TMA(128, 128, 16, 64, 32, 4),
    DG_TMA(128, 128, 16, 32, 64, 4),
    DG_TMA(128, 128, 16, 32, 32, 4),
    DG_TMA(128, 128, 32, 64, 32, 3),
    DG_TMA(128, 128, 32, 32, 32, 3),
    DG_TMA(128, 128, 16, 64, 32, 6),
    DG_TMA(128, 128, 16, 32, 32, 6),
    DG_TMA(256, 64, 16, 64, 32, 4),
    DG_TMA(256, 64, 16, 32, 32, 4),
    DG_TMA_XP(256, 64, 16, 64, 32, 4),
    DG_TMA_XP(128, 128, 16, 64, 32, 4),
    DG_HYB(256, 64, 16, 64, 32, 4),
};

const CfgEntry *cfg_table_big(int *n) {
    *n = (int)(sizeof(k_table) / sizeof(k_table[0]));
    return k_table;
}

}  // namespace dg
