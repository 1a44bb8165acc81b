// cfgs_generic.cu -- cp.async configurations (any alignment / odd leading dimensions).
#include "registry.cuh"

namespace dg {

static const CfgEntry k_table[] = {
    DG_GEN(128, 128, 16, 64, 32, 4),
    DG_GEN(64, 64, 16, 32, 16, 4),
};

const CfgEntry *cfg_table_generic(int *n) {
    *n = (int)(sizeof(k_table) / sizeof(k_table[0]));
    return k_table;
}

}  // namespace dg
