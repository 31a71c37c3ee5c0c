// tiles.cuh — the tiled fp32 copy S_t of the score matrix consumed by the tensor-core SYRK.
//
// S (n x m, row-major, 4 MB row pitch at m = 1e6) is a poor TMA source: a 128-row x 128-byte
// operand box is 128 separate strided row requests (measured 16 B/clk/SM, tools/ubench/
// tma_rows.cu).  The u = S v streaming pass therefore also writes S_t, in which every
// 128-row x 32-column tile is one contiguous 16 KB block already in the SWIZZLE_128B shared-
// memory image the tcgen05 descriptors expect, so the SYRK moves it with one 1-D bulk copy.
//   tile (kb, rb) at byte offset ((kb * nb) + rb) * 16 KB   (kb = K-block, rb = 128-row block)
//   element (r, c) of a tile at r * 128 + (((c >> 2) ^ (r & 7)) << 4) + (c & 3) * 4
// Rows >= n and columns >= m of the padded extent (even block count) are zero.
#pragma once
#include <stdint.h>

namespace fs {
constexpr int kTileRows = 128;
constexpr int kTileCols = 32;
constexpr int kTileBytes = kTileRows * kTileCols * 4;

// row blocks, rounded up to an even count: the SYRK's CTA pairs always read blocks 2p and 2p+1
__host__ __device__ inline int64_t tiles_nb(int64_t n) { return ((n + 2 * kTileRows - 1) / (2 * kTileRows)) * 2; }
__host__ __device__ inline int64_t tiles_kb(int64_t m) { return (m + kTileCols - 1) / kTileCols; }
__host__ __device__ inline size_t tiles_bytes(int64_t n, int64_t m) {
  return (size_t)tiles_nb(n) * tiles_kb(m) * kTileBytes;
}
// byte offset of the 16-byte chunk holding columns 4*chunk..4*chunk+3 of row i, K-block kb
__host__ __device__ inline size_t tile_chunk_offset(int64_t nb, int64_t kb, int64_t i, int chunk) {
  const int r = (int)(i & (kTileRows - 1));
  return ((size_t)kb * nb + (size_t)(i >> 7)) * kTileBytes + (size_t)r * 128 + (size_t)((chunk ^ (r & 7)) << 4);
}

// ---- F16X2 split copy: per row i a power-of-two scale s_i (fs.h FS_PREC_F16X2); every
// element is stored as hi = fp16_rn(x s_i) and lo = fp16_rn(x s_i - hi) in two planes.  A tile
// is 128 rows x 64 columns (128-byte fp16 rows, SWIZZLE_128B image); the hi and lo tiles of a
// (K-block, row block) are adjacent, so one 32 KB bulk copy moves both:
//   plane p of tile (kb, rb) at byte offset (((kb * nb) + rb) * 2 + p) * 16 KB
//   element (r, c) at r * 128 + (((c >> 3) ^ (r & 7)) << 4) + (c & 7) * 2
constexpr int kTile16Cols = 64;
__host__ __device__ inline int64_t tiles16_kb(int64_t m) { return (m + kTile16Cols - 1) / kTile16Cols; }
__host__ __device__ inline size_t tiles16_bytes(int64_t n, int64_t m) {
  return (size_t)tiles_nb(n) * tiles16_kb(m) * 2 * kTileBytes;
}
// byte offset of the 16-byte chunk holding columns 8*chunk..8*chunk+7 of row i, K-block kb, plane p
__host__ __device__ inline size_t tile16_chunk_offset(int64_t nb, int64_t kb, int64_t i, int chunk, int plane) {
  const int r = (int)(i & (kTileRows - 1));
  return (((size_t)kb * nb + (size_t)(i >> 7)) * 2 + plane) * kTileBytes + (size_t)r * 128 +
         (size_t)((chunk ^ (r & 7)) << 4);
}
}  // namespace fs
