// Fused single-pass forward scan (fast path).  Stub: not yet enabled.
#pragma once
#include "k_scan_fwd.cuh"

namespace pdssm {

inline size_t fused_ws_bytes(int64_t S, int C) {
    (void)S;
    (void)C;
    return 0;
}

inline pdssm_status fwd_fused_try(int64_t, int64_t, int64_t, int64_t, int64_t, int, int, int, int, int, uint32_t,
                                  const uint8_t*, const uint16_t*, const uint16_t*, const uint16_t*, const void*,
                                  const void*, const float*, ChunkStateView, uint16_t*, void*, void*, cudaStream_t,
                                  bool* done) {
    *done = false;
    return PDSSM_OK;
}

}  // namespace pdssm
