// Instantiations of the field-walk search kernel (QB_VARIANT_FIELDWALK, large-block geometry).
#include "qb_fieldwalk.cuh"
#include "qb_registry.h"

namespace qb {

static_assert(BIG_BE == FW_RB, "field-walk reporting blocks must match the table blocks");
#define QB_F(L) LFn { L, fieldwalk_kernel<L, TPB>, nullptr }
static const LFn kFieldwalk[] = {QB_F(11), QB_F(12), QB_F(13), QB_F(14), QB_F(16), QB_F(18), QB_F(20), QB_F(22)};

const LFn* fieldwalk_fns(int* count) {
  *count = (int)(sizeof(kFieldwalk) / sizeof(kFieldwalk[0]));
  return kFieldwalk;
}

}  // namespace qb
