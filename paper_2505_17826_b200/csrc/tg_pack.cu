// tg_pack.cu -- on-device experience packer.
//
// Turns a padded token batch ([B, L] ids + loss mask, optional dense old / ref
// logprobs aligned to the ids) into the packed row layout of tg_loss.h with the
// HF shift applied: trainable row for target position (b, l), l >= 1 and
// mask[b, l] != 0, reads logits row (b, l - 1) of the [B * L, V] logits (via
// row_index -- no gather copy) and scores target ids[b, l].  Rows keep the
// (b, l) order, so sequences are contiguous and in batch order, as
// ExperienceBuffer.sample_batch returns them (buffer.py:251-264); interior
// mask-false spans (multi-turn environment / role tokens, workflows.py:128-183)
// are compacted out.  The reference's compact per-experience logprob list
// (records.py:47-49) is exactly `old_lp` in this order.
//
//   k_pack_count  warp per sequence: trainable rows per sequence
//   k_pack_scan   one CTA: exclusive scan -> seq_offsets[B+1], total rows
//   k_pack_emit   warp per sequence: ballot / popc compaction of the positions
#include <stdint.h>

#include "tg_common.cuh"

namespace tg {

struct PackParams {
  const uint8_t* mask;   // [B * L]
  const void* ids;       // [B * L] int32 or int64
  int ids64;
  const float* old_dense;  // optional [B * L]
  const float* ref_dense;  // optional [B * L]
  int32_t B, L;
  int64_t* row_index;    // [cap]
  int32_t* target;       // [cap]
  float* old_out;        // optional [cap]
  float* ref_out;        // optional [cap]
  int32_t* seq_offsets;  // [B + 1]
  int32_t* counts;       // [B] workspace
  int64_t* n_rows;       // [1] device
  int64_t cap;
};

__device__ __forceinline__ bool trainable(const PackParams& p, int b, int l) {
  return l >= 1 && p.mask[int64_t(b) * p.L + l] != 0;
}

__global__ void k_pack_count(const PackParams p) {
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= p.B) return;
  int n = 0;
  for (int l = lane; l < p.L; l += 32) n += trainable(p, b, l) ? 1 : 0;
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) n += __shfl_xor_sync(0xffffffffu, n, d);
  if (lane == 0) p.counts[b] = n;
}

// single CTA, 1024 threads: sequential-block exclusive scan (B is small)
__global__ void k_pack_scan(const PackParams p) {
  __shared__ int64_t part[1024];
  const int tid = threadIdx.x;
  const int per = (p.B + 1023) / 1024;
  const int b0 = tid * per, b1 = min(p.B, b0 + per);
  int64_t s = 0;
  for (int b = b0; b < b1; ++b) s += p.counts[b];
  part[tid] = s;
  __syncthreads();
  if (tid == 0) {
    int64_t acc = 0;
    for (int i = 0; i < 1024; ++i) {
      const int64_t v = part[i];
      part[i] = acc;
      acc += v;
    }
    *p.n_rows = acc;
    p.seq_offsets[p.B] = int32_t(acc);
  }
  __syncthreads();
  int64_t o = part[tid];
  for (int b = b0; b < b1; ++b) {
    p.seq_offsets[b] = int32_t(o);
    o += p.counts[b];
  }
}

__global__ void k_pack_emit(const PackParams p) {
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= p.B) return;
  int64_t out = p.seq_offsets[b];
  for (int l0 = 0; l0 < p.L; l0 += 32) {
    const int l = l0 + lane;
    const bool t = l < p.L && trainable(p, b, l);
    const uint32_t bal = __ballot_sync(0xffffffffu, t);
    if (t) {
      const int64_t r = out + __popc(bal & ((1u << lane) - 1u));
      if (r < p.cap) {
        const int64_t pos = int64_t(b) * p.L + l;
        p.row_index[r] = pos - 1;  // HF shift: logits at l - 1 score token l
        p.target[r] = p.ids64 ? int32_t(reinterpret_cast<const int64_t*>(p.ids)[pos])
                              : reinterpret_cast<const int32_t*>(p.ids)[pos];
        if (p.old_out) p.old_out[r] = p.old_dense ? p.old_dense[pos] : 0.f;
        if (p.ref_out) p.ref_out[r] = p.ref_dense ? p.ref_dense[pos] : 0.f;
      }
    }
    out += __popc(bal);
  }
}

}  // namespace tg

using namespace tg;

extern "C" int tg_pack_rows(const uint8_t* mask, const void* ids, int ids_is_int64, int32_t B,
                            int32_t L, const float* old_dense, const float* ref_dense,
                            int64_t* row_index, int32_t* target, float* old_out, float* ref_out,
                            int64_t capacity, int32_t* seq_offsets, int64_t* n_rows,
                            void* workspace, size_t workspace_bytes, void* stream) {
  if (B < 0 || L < 0 || !seq_offsets || !n_rows || (B > 0 && (!mask || !ids || !workspace)))
    return TG_EINVAL;
  if (workspace_bytes < size_t(B) * 4) return TG_EWORKSPACE;
  if (capacity > 0 && (!row_index || !target)) return TG_EINVAL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  PackParams p;
  p.mask = mask;
  p.ids = ids;
  p.ids64 = ids_is_int64;
  p.old_dense = old_dense;
  p.ref_dense = ref_dense;
  p.B = B;
  p.L = L;
  p.row_index = row_index;
  p.target = target;
  p.old_out = old_out;
  p.ref_out = ref_out;
  p.seq_offsets = seq_offsets;
  p.counts = reinterpret_cast<int32_t*>(workspace);
  p.n_rows = n_rows;
  p.cap = capacity;
  cudaGetLastError();
  if (B > 0) k_pack_count<<<(B + 7) / 8, 256, 0, st>>>(p);
  k_pack_scan<<<1, 1024, 0, st>>>(p);
  if (B > 0) k_pack_emit<<<(B + 7) / 8, 256, 0, st>>>(p);
  return cudaGetLastError() == cudaSuccess ? TG_OK : TG_ECUDA;
}
