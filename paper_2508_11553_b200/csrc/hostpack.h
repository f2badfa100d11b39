// Host side of the packed host->device token copy.
//
// Token ids from host buffers cross PCIe as 18-bit split planes: a uint16 low plane
// (one entry per position) and a 2-bit high plane (one byte per 4 positions; byte j of a
// 32-position group holds positions j, j+8, j+16, j+24 at bits 0, 2, 4, 6).  2.25 B per
// token instead of 4; k_unpack18 restores int32 words on the device.  Packing runs on a
// pool of host threads with non-temporal stores, chunk by chunk, while the copy engine
// moves the previous chunk.  Any id outside [0, 2^18) makes the caller fall back to the
// raw int32 copy.
#pragma once
#include <cstdint>
#include <functional>

namespace tms {

struct PackPiece {
  const int32_t *src;  // caller's tokens
  int64_t dst;         // destination position (multiple of 32)
  int64_t len;         // tokens
};

constexpr int64_t kPackPieceMax = 1 << 15;  // tokens per piece (work unit of one pool thread)

bool pack18_supported();
// Pack one piece into lo / hi (non-temporal stores, fenced); false if any token is
// outside [0, 2^18).
bool pack_piece(const PackPiece &p, uint16_t *lo, uint8_t *hi);
// memcpy with non-temporal stores (no read-for-ownership of the destination): for large
// pinned -> pageable copies of results; falls back to memcpy without AVX2.
void copy_stream(void *dst, const void *src, size_t n);
// Host thread pool shared by all stores of the process (TM_HOST_THREADS, default: all cores
// up to 16).
int host_threads();
void parallel_for(int64_t n, const std::function<void(int64_t)> &fn);

}  // namespace tms
