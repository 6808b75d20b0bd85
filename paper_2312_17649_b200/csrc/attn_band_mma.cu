// Placeholder: tiled band kernel arrives in the next commit.
#include "attn.cuh"
namespace sc {
size_t band_workspace_bytes(int, int, int, int, int) { return 0; }
int launch_attn_band(const AttnArgs&, int, const int32_t*, const int32_t*, int, void*, size_t,
                     cudaStream_t) {
  set_error("band kernel not built");
  return SC_ERR_UNSUPPORTED;
}
}  // namespace sc
