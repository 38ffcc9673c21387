// bf16 tcgen05/TMEM query path (placeholder until the tensor-core kernel lands).
#include "nasg_internal.h"

namespace nasg {
bool tc_supported(int) { return false; }
size_t tc_image_bytes(int) { return 0; }
void launch_pack_tc(const float *, int, void *, cudaStream_t) {}
int query_tc(int, QueryMode, const void *, const QueryArgs &, int, cudaStream_t) { return -1; }
}  // namespace nasg
