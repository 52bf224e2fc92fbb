// Instantiations of the table-kernel family (search, collect stages, prefix hook).
#include "qb_registry.h"
#include "qb_table.cuh"

namespace qb {

#define QB_T(B1, B2, L)                                                                                  \
  TableFns {                                                                                             \
    B1, B2, L, table_kernel<B1, B2, 0, L, TPB>, collect_mark_kernel<B1, B2, 0, L>,                       \
        collect_blocks_kernel<B1, B2, 0, L>, collect_states_kernel<B1, B2, 0, L>,                        \
        prefix_eval_kernel<B1, B2, 0, L>                                                                 \
  }

// small problems: one block of 2^L states per chunk (L = block bits <= 10); large problems: 10-bit
// blocks, L free bits per chunk
static const TableFns kTable[] = {
    QB_T(0, 1, 1),  QB_T(1, 1, 2),  QB_T(1, 2, 3),  QB_T(2, 2, 4),  QB_T(2, 3, 5),  QB_T(3, 3, 6),
    QB_T(3, 4, 7),  QB_T(4, 4, 8),  QB_T(4, 5, 9),  QB_T(BIG_B1, BIG_B2, 10),
    QB_T(BIG_B1, BIG_B2, 11), QB_T(BIG_B1, BIG_B2, 12), QB_T(BIG_B1, BIG_B2, 13), QB_T(BIG_B1, BIG_B2, 14),
    QB_T(BIG_B1, BIG_B2, 16), QB_T(BIG_B1, BIG_B2, 18), QB_T(BIG_B1, BIG_B2, 20), QB_T(BIG_B1, BIG_B2, 22),
};

const TableFns* table_fns(int* count) {
  *count = (int)(sizeof(kTable) / sizeof(kTable[0]));
  return kTable;
}

}  // namespace qb
