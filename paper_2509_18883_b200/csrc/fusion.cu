// Task-vector fusion kernels for sm_100a (K1 norm partials, finalize, K2 dropout bitmap, K3 merge).
//
// Reference algorithm (pkg/src/rolloutlab/fusion.py):
//   task_vector           79-83    delta = expert - base (f64, exact for bf16/f32 inputs)
//   TaskVector.norm       37-44    ||delta||_2
//   normalize_magnitudes  86-102   target = mean of non-zero norms | fixed | None; delta * (target / norm)
//   dropout_prune        105-115   keep iff uniform >= p (SplitMix64 stream rng.split(i)), survivors / (1 - p)
//   erase_minority       118-142   majority = sign(sum_i k_i) or sign(sum_i sign(k_i) k_i^2); zero opposers
//   fuse                 154-188   fused = base; fused = fused + w_i * k_i (sequential), FusionStats
//
// Both passes are persistent, warp-specialised TMA pipelines: one producer warp issues 1-D bulk
// copies (cp.async.bulk -> SASS UBLKCP) of every stream's stage tile into a shared-memory ring,
// completion tracked by mbarrier transaction counts; eight consumer warps read the stage with 128-bit
// LDS, compute, and release the slot.  Grid = one CTA per SM, items strided over CTAs.
#include "common.cuh"
#include "capi_internal.h"
#include "pipeline.cuh"

namespace rlk {

constexpr uint32_t kItem = RLK_FUSION_ITEM;
constexpr uint32_t kSmemBudget = 210 * 1024;

template <int N> struct StreamBytes { static constexpr uint32_t v = N <= 4 ? 8192u : 4096u; };

struct ItemGeom {
  const rlk_fusion_segment* seg;
  uint64_t j0;  // seg->j0 (cached)
  void* out;    // seg->out (cached)
  uint64_t start;  // element offset of the item within its piece
  uint32_t len;
  uint32_t gitem;
  uint32_t tensor;
};

// Items of a CTA are visited in increasing order (item += gridDim.x) and segments are in item order,
// so the segment of the next item is found by a forward scan from the current one, and the
// segment's fields are re-read only when it changes: one item's geometry costs no global loads in
// the common case, instead of a dependent binary search (~log2(n_segs) L2 round trips) per item.
struct SegCursor {
  uint32_t lo = 0xffffffffu;  // current segment (none yet)
  uint32_t p_lo = 0, p_hi = 0;  // seg_item_prefix[lo], seg_item_prefix[lo + 1]
  const rlk_fusion_segment* seg = nullptr;
  uint64_t numel = 0, j0 = 0;
  void* out = nullptr;
  uint32_t item0 = 0, tensor = 0;
  // moves to the segment holding `item`; returns true when it changed
  __device__ __forceinline__ bool seek(const rlk_fusion_plan& plan, uint32_t item) {
    if (lo != 0xffffffffu && item < p_hi) return false;
    if (lo == 0xffffffffu) {
      lo = 0;
      p_lo = __ldg(plan.seg_item_prefix);
      p_hi = __ldg(plan.seg_item_prefix + 1);
    }
    while (item >= p_hi) {
      ++lo;
      p_lo = p_hi;
      p_hi = __ldg(plan.seg_item_prefix + lo + 1);
    }
    seg = plan.segs + lo;
    numel = seg->numel;
    j0 = seg->j0;
    out = seg->out;
    item0 = seg->item0;
    tensor = seg->tensor;
    return true;
  }
};

__device__ __forceinline__ ItemGeom item_geom_bs(const rlk_fusion_plan& plan, uint32_t item) {
  uint32_t lo = 0, hi = plan.n_segs;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(plan.seg_item_prefix + mid) <= item) lo = mid; else hi = mid;
  }
  ItemGeom g;
  g.seg = plan.segs + lo;
  g.j0 = g.seg->j0;
  g.out = g.seg->out;
  uint32_t k = item - __ldg(plan.seg_item_prefix + lo);
  g.start = (uint64_t)k * kItem;
  uint64_t rem = g.seg->numel - g.start;
  g.len = rem < kItem ? (uint32_t)rem : kItem;
  g.gitem = g.seg->item0 + k;
  g.tensor = g.seg->tensor;
  return g;
}

__device__ __forceinline__ ItemGeom item_geom(const rlk_fusion_plan& plan, SegCursor& c, uint32_t item) {
  c.seek(plan, item);
  ItemGeom g;
  g.seg = c.seg;
  g.j0 = c.j0;
  g.out = c.out;
  const uint32_t k = item - c.p_lo;
  g.start = (uint64_t)k * kItem;
  const uint64_t rem = c.numel - g.start;
  g.len = rem < kItem ? (uint32_t)rem : kItem;
  g.gitem = c.item0 + k;
  g.tensor = c.tensor;
  return g;
}

// Producer: one elected lane streams every (item, stage) of this CTA through the ring.
// Stage layout: [stream 0 | stream 1 | ... | stream NS-1 | bitmap expert 0 | ... | bitmap expert N-1].
// kCursor: item geometry from the incremental SegCursor (K3: its per-item stalls cost bandwidth) or a
// binary search per item (K1: measured faster there, same-box A/B)
template <int ESZ, int N, uint32_t SB = StreamBytes<N>::v, bool kCursor = true>
__device__ void produce(const rlk_fusion_plan& plan, const Ring& r, bool with_base, const uint32_t* bitmap,
                        uint64_t words_per_row, uint32_t sub_shift = 0) {
  constexpr uint32_t ELEMS = SB / ESZ;
  constexpr uint32_t BMB = ELEMS / 8;  // bitmap bytes per expert per full stage
  const int ns = with_base ? N + 1 : N;
  // parameter streams are read once (evict_first); every tensor re-reads the keep-bitmap prefix
  // [0, numel) of each expert row, so the bitmap is kept in L2 (evict_last): the prefixes of all but
  // the embedding-sized tensors fit, and their re-reads stop costing HBM traffic
  const uint64_t pol = policy_evict_first();
  const uint64_t pol_bm = policy_evict_last();
  RingPos q;
  SegCursor cur;
  const uint32_t unit = kItem >> sub_shift;
  for (uint32_t u = blockIdx.x; u < (plan.n_items << sub_shift); u += gridDim.x) {
    const uint32_t item = u >> sub_shift;
    const ItemGeom g = kCursor ? item_geom(plan, cur, item) : item_geom_bs(plan, item);
    const uint32_t lo = (u & ((1u << sub_shift) - 1u)) * unit;  // the unit's element range [lo, hi)
    if (lo >= g.len) continue;
    const uint32_t hi = min(g.len, lo + unit);
    const char* src[N + 1];
    if (!with_base) {
#pragma unroll
      for (int i = 0; i < N; ++i) src[i] = (const char*)g.seg->expert[i];
    } else {
      src[0] = (const char*)g.seg->base;
#pragma unroll
      for (int i = 0; i < N; ++i) src[i + 1] = (const char*)g.seg->expert[i];
    }
    const uint64_t jtensor0 = g.j0 + g.start;
    for (uint32_t off = lo; off < hi; off += ELEMS) {
      const uint32_t n = min(ELEMS, hi - off);
      const uint32_t main_bytes = (n * ESZ) & ~15u;
      const uint32_t bm_bytes = bitmap ? (((n + 7) / 8 + 15) & ~15u) : 0u;
      const uint32_t s = q.s, ph = q.ph;
      mbar_wait(&r.empty[s], ph ^ 1u);
      const uint32_t tx = main_bytes * ns + bm_bytes * N;
      uint8_t* dst = r.buf + s * r.stage_bytes;
      RLK_DCHECK(s < r.nstages && off + n <= hi && hi <= g.len && g.start + g.len <= g.seg->numel);
      RLK_DCHECK(main_bytes <= SB && ns * SB <= r.stage_bytes);
      RLK_DCHECK(!bitmap || ((N + 1) * SB + N * BMB <= r.stage_bytes && bm_bytes <= BMB));
      RLK_DCHECK(!bm_bytes || (jtensor0 + off) / 8 + bm_bytes <= words_per_row * 4);
      if (tx) {
        mbar_arrive_expect_tx(&r.full[s], tx);
        if (main_bytes) {
          const uint64_t byte_off = (g.start + off) * ESZ;
          for (int k = 0; k < ns; ++k) bulk_g2s(dst + k * SB, src[k] + byte_off, main_bytes, &r.full[s], pol);
        }
        if (bm_bytes) {
          const uint64_t jb = jtensor0 + off;  // multiple of ELEMS -> byte offset multiple of 16
          for (int i = 0; i < N; ++i)
            bulk_g2s(dst + (N + 1) * SB + i * BMB, (const char*)(bitmap + i * words_per_row) + jb / 8, bm_bytes,
                     &r.full[s], pol_bm);
        }
      } else {
        mbar_arrive(&r.full[s]);
      }
      q.next(r.nstages);
    }
  }
}

// ------------------------------------------------------------------ vector unpack helpers
template <int DT> struct VecIO;
template <> struct VecIO<RLK_BF16> {
  static constexpr int n = 8;
  __device__ static void f32(const uint4& w, float* o) {
    o[0] = bf16_lo(w.x); o[1] = bf16_hi(w.x); o[2] = bf16_lo(w.y); o[3] = bf16_hi(w.y);
    o[4] = bf16_lo(w.z); o[5] = bf16_hi(w.z); o[6] = bf16_lo(w.w); o[7] = bf16_hi(w.w);
  }
  __device__ static void f64(const uint4& w, double* o) {
    float t[8];
    f32(w, t);
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = (double)t[e];
  }
};
template <> struct VecIO<RLK_F32> {
  static constexpr int n = 4;
  __device__ static void f64(const uint4& w, double* o) {
    o[0] = (double)__uint_as_float(w.x); o[1] = (double)__uint_as_float(w.y);
    o[2] = (double)__uint_as_float(w.z); o[3] = (double)__uint_as_float(w.w);
  }
};
template <> struct VecIO<RLK_F64> {
  static constexpr int n = 2;
  __device__ static void f64(const uint4& w, double* o) {
    o[0] = __hiloint2double((int)w.y, (int)w.x);
    o[1] = __hiloint2double((int)w.w, (int)w.z);
  }
};

// Store VEC outputs (given as f64) at element index idx of out (vectorised when aligned).
template <int DTO, int VEC>
__device__ __forceinline__ void store_vec_f64(void* out, uint64_t idx, const double* y) {
  if constexpr (DTO == RLK_BF16) {
    uint32_t h[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) h[e] = f64_to_bf16_rne(y[e]);
    if constexpr (VEC == 8) {
      uint4 w = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
      stg128_stream((uint16_t*)out + idx, w);
    } else if constexpr (VEC == 4) {
      *reinterpret_cast<uint2*>((uint16_t*)out + idx) = make_uint2(h[0] | (h[1] << 16), h[2] | (h[3] << 16));
    } else {
      *reinterpret_cast<uint32_t*>((uint16_t*)out + idx) = h[0] | (h[1] << 16);
    }
  } else if constexpr (DTO == RLK_F32) {
    float f[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) f[e] = f64_to_f32_rn(y[e]);
#pragma unroll
    for (int e = 0; e < VEC; e += 4) {
      if constexpr (VEC >= 4) {
        stg128_stream((float*)out + idx + e, make_uint4(__float_as_uint(f[e]), __float_as_uint(f[e + 1]),
                                                         __float_as_uint(f[e + 2]), __float_as_uint(f[e + 3])));
      }
    }
    if constexpr (VEC == 2) *reinterpret_cast<float2*>((float*)out + idx) = make_float2(f[0], f[1]);
  } else {
#pragma unroll
    for (int e = 0; e < VEC; e += 2) {
      stg128_stream((double*)out + idx + e,
                    make_uint4(__double2loint(y[e]), __double2hiint(y[e]), __double2loint(y[e + 1]),
                               __double2hiint(y[e + 1])));
    }
  }
}

// ------------------------------------------------------------------ K1: norm partials (+ non-zero counts)
struct SumsqArgs {
  rlk_fusion_plan plan;
  double* partials;
  unsigned long long* counters;  // nullable: [t*2N + i] += non-zero entries after dropout
  const uint32_t* bitmap;        // dropout_mode 2
  uint64_t words_per_row;
  uint64_t seed[RLK_MAX_EXPERTS];
  uint64_t thresh;
  int delta_mode, dropout_mode;
  uint32_t stage_bytes, nstages;
};

// Two CTAs per SM: the loop is bound by F2F (XU pipe) and fp64 latency, so it needs the warps.
// CM >= 0 (f32 pair mode): the counting mode fixed at compile time -- 0 no counters, 1 every entry
// kept, 2 keep bits from the K2 bitmap -- and the non-zero test done on the f32 inputs (x != b; the
// inputs are finite whenever the counts are used: non-finite norms fail the call).
template <int DT, int N, int CM = -1>
__global__ void __launch_bounds__(kThreads, 2) k_sumsq(const __grid_constant__ SumsqArgs a) {
  static_assert(CM < 0 || DT == RLK_F32, "compile-time counting mode: f32 pair mode only");
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int ESZ = Elem<DT>::size;
  constexpr int VEC = 16 / ESZ;
  constexpr uint32_t SB = StreamBytes<N>::v;
  constexpr uint32_t ELEMS = SB / ESZ;
  constexpr uint32_t BMB = ELEMS / 8;
  const Ring r = ring_setup(smem, a.stage_bytes, a.nstages);
  const bool delta = CM >= 0 ? false : a.delta_mode != 0;
  const bool count = CM >= 0 ? CM != 0 : a.counters != nullptr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == kCWarps) {
    if (lane == 0) produce<ESZ, N, StreamBytes<N>::v, false>(a.plan, r, !delta, (count && a.dropout_mode == 2) ? a.bitmap : nullptr,
                                   a.words_per_row);
    return;
  }
  __shared__ double red[kCWarps][N];
  const int tid = threadIdx.x;
  RingPos q;
  SegCursor cur;
  for (uint32_t item = blockIdx.x; item < a.plan.n_items; item += gridDim.x) {
    const ItemGeom g = item_geom(a.plan, cur, item);
    const uint64_t jtensor0 = g.j0 + g.start;
    double acc[N][2];
    uint32_t nz[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      acc[i][0] = acc[i][1] = 0.0;
      nz[i] = 0;
    }
    for (uint32_t off = 0; off < g.len; off += ELEMS) {
      const uint32_t n = min(ELEMS, g.len - off);
      const uint32_t main_elems = ((n * ESZ) & ~15u) / ESZ;
      const uint32_t s = q.s, ph = q.ph;
      mbar_wait(&r.full[s], ph);
      const uint8_t* sb = r.buf + s * r.stage_bytes;
      const uint8_t* bm = sb + (N + 1) * SB;
      const uint32_t nvec = main_elems / VEC;
      for (uint32_t v = tid; v < nvec; v += kCThreads) {
        const uint32_t le = v * VEC;
        if constexpr (CM >= 0) {
          const uint4 bq = lds128(sb + v * 16);
          double b[4];
          VecIO<RLK_F32>::f64(bq, b);
#pragma unroll
          for (int i = 0; i < N; ++i) {
            const uint4 xq = lds128(sb + (i + 1) * SB + v * 16);
            double x[4];
            VecIO<RLK_F32>::f64(xq, x);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const double d = x[e] - b[e];
              acc[i][e & 1] = fma(d, d, acc[i][e & 1]);
            }
            if constexpr (CM != 0) {
              const uint32_t neq = (uint32_t)(__uint_as_float(xq.x) != __uint_as_float(bq.x)) |
                                   (uint32_t)(__uint_as_float(xq.y) != __uint_as_float(bq.y)) << 1 |
                                   (uint32_t)(__uint_as_float(xq.z) != __uint_as_float(bq.z)) << 2 |
                                   (uint32_t)(__uint_as_float(xq.w) != __uint_as_float(bq.w)) << 3;
              const uint32_t keep = CM == 2 ? (uint32_t)(bm[i * BMB + (le >> 3)] >> (le & 7)) : 0xfu;
              nz[i] += __popc(neq & keep & 0xfu);
            }
          }
          continue;
        }
        double b[VEC];
        if (!delta) VecIO<DT>::f64(lds128(sb + v * 16), b);
        else {
#pragma unroll
          for (int e = 0; e < VEC; ++e) b[e] = 0.0;
        }
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double x[VEC];
          VecIO<DT>::f64(lds128(sb + (i + (delta ? 0 : 1)) * SB + v * 16), x);
          uint32_t keep = (1u << VEC) - 1u;
          if (count && a.dropout_mode == 2) {
            keep = (bm[i * BMB + (le >> 3)] >> (le & 7)) & ((1u << VEC) - 1u);
          } else if (count && a.dropout_mode == 1) {
            keep = 0;
#pragma unroll
            for (int e = 0; e < VEC; ++e) keep |= (uint32_t)keep_draw(a.seed[i], jtensor0 + off + le + e, a.thresh) << e;
          }
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const double d = delta ? x[e] : x[e] - b[e];
            acc[i][e & 1] = fma(d, d, acc[i][e & 1]);
            if (count) nz[i] += ((keep >> e) & 1u) && (d != 0.0);
          }
        }
      }
      for (uint32_t e = main_elems + tid; e < n; e += kCThreads) {
        const uint64_t idx = g.start + off + e;
        const double b = delta ? 0.0 : load_f64<DT>(g.seg->base, idx);
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const double x = load_f64<DT>(g.seg->expert[i], idx);
          const double d = delta ? x : x - b;
          acc[i][0] = fma(d, d, acc[i][0]);
          if (count) {
            const bool keep = a.dropout_mode == 0 || keep_draw(a.seed[i], jtensor0 + off + e, a.thresh);
            nz[i] += keep && (d != 0.0);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&r.empty[s]);
      q.next(r.nstages);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double w = warp_sum_f64(acc[i][0] + acc[i][1]);
      if (lane == 0) red[warp][i] = w;
      if (count) {
        const uint32_t z = __reduce_add_sync(0xffffffffu, nz[i]);
        if (lane == 0 && z) atomicAdd(a.counters + (uint64_t)g.tensor * 2 * N + i, (unsigned long long)z);
      }
    }
    cbar_sync();
    if (tid < N) {
      double t = red[0][tid];
#pragma unroll
      for (int w = 1; w < kCWarps; ++w) t += red[w][tid];
      a.partials[(uint64_t)g.gitem * N + tid] = t;
    }
    cbar_sync();
  }
}

// K1 for bf16 pair-mode inputs: exact f64 squares of (expert - base) with the bf16 -> f64 widening
// done once for the base and once per expert (F2F on the XU pipe), two independent f64 accumulator
// chains per expert, and the non-zero-after-dropout count as popc(neq_bits & keep_bits) per vector.
// COUNT: 0 no counting, 1 no dropout (every entry kept), 2 keep bits from the K2 bitmap.
template <int N, int COUNT>
__global__ void __launch_bounds__(kThreads, 2) k_sumsq_bf16(const __grid_constant__ SumsqArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr uint32_t SB = StreamBytes<N>::v;
  constexpr uint32_t ELEMS = SB / 2;
  constexpr uint32_t BMB = ELEMS / 8;
  const Ring r = ring_setup(smem, a.stage_bytes, a.nstages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == kCWarps) {
    if (lane == 0) produce<2, N, StreamBytes<N>::v, false>(a.plan, r, true, COUNT == 2 ? a.bitmap : nullptr, a.words_per_row);
    return;
  }
  __shared__ double red[kCWarps][N];
  const int tid = threadIdx.x;
  RingPos q;
  for (uint32_t item = blockIdx.x; item < a.plan.n_items; item += gridDim.x) {
        const ItemGeom g = item_geom_bs(a.plan, item);
    const uint64_t jtensor0 = g.j0 + g.start;
    double acc0[N], acc1[N];
    uint32_t nz[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      acc0[i] = acc1[i] = 0.0;
      nz[i] = 0;
    }
    for (uint32_t off = 0; off < g.len; off += ELEMS) {
      const uint32_t n = min(ELEMS, g.len - off);
      const uint32_t main_elems = ((n * 2) & ~15u) / 2;
      const uint32_t s = q.s, ph = q.ph;
      mbar_wait(&r.full[s], ph);
      const uint8_t* sb = r.buf + s * r.stage_bytes;
      const uint8_t* bm = sb + (N + 1) * SB;
      const uint32_t nvec = main_elems / 8;
      for (uint32_t v = tid; v < nvec; v += kCThreads) {
        float bf[8];
        VecIO<RLK_BF16>::f32(lds128(sb + v * 16), bf);
        double bd[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) bd[e] = (double)bf[e];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          float xf[8];
          VecIO<RLK_BF16>::f32(lds128(sb + (i + 1) * SB + v * 16), xf);
          uint32_t neq = 0;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const double d = (double)xf[e] - bd[e];
            if (e & 1) acc1[i] = fma(d, d, acc1[i]);
            else acc0[i] = fma(d, d, acc0[i]);
            if (COUNT) neq |= (xf[e] != bf[e]) ? (1u << e) : 0u;
          }
          if (COUNT == 1) nz[i] += __popc(neq);
          if (COUNT == 2) nz[i] += __popc(neq & (uint32_t)bm[i * BMB + v]);
        }
      }
      for (uint32_t e = main_elems + tid; e < n; e += kCThreads) {
        const uint64_t idx = g.start + off + e;
        const double b = load_f64<RLK_BF16>(g.seg->base, idx);
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const double d = load_f64<RLK_BF16>(g.seg->expert[i], idx) - b;
          acc0[i] = fma(d, d, acc0[i]);
          if (COUNT) {
            const bool keep = COUNT == 1 || keep_draw(a.seed[i], jtensor0 + off + e, a.thresh);
            nz[i] += keep && (d != 0.0);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&r.empty[s]);
      q.next(r.nstages);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double w = warp_sum_f64(acc0[i] + acc1[i]);
      if (lane == 0) red[warp][i] = w;
      if (COUNT) {
        const uint32_t z = __reduce_add_sync(0xffffffffu, nz[i]);
        if (lane == 0 && z) atomicAdd(a.counters + (uint64_t)g.tensor * 2 * N + i, (unsigned long long)z);
      }
    }
    cbar_sync();
    if (tid < N) {
      double t = red[0][tid];
#pragma unroll
      for (int w = 1; w < kCWarps; ++w) t += red[w][tid];
      a.partials[(uint64_t)g.gitem * N + tid] = t;
    }
    cbar_sync();
  }
}

// ------------------------------------------------------------------ finalize: norms -> scales
// One warp per tensor; lane l sums items l, l+32, ... then a fixed xor-tree: the result depends only
// on the global item partition, never on which rank produced which partial.
__global__ void k_finalize(const double* __restrict__ partials, const uint32_t* __restrict__ tensor_items,
                           uint32_t n_tensors, int n, int target_mode, double target_value,
                           double* __restrict__ sumsq, double* __restrict__ scale, int32_t* __restrict__ status) {
  const uint32_t t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= n_tensors) return;
  const uint32_t i0 = tensor_items[t], i1 = tensor_items[t + 1];
  double norms[RLK_MAX_EXPERTS];
  bool finite = true;
  for (int i = 0; i < n; ++i) {
    double acc = 0.0;
    for (uint32_t k = i0 + lane; k < i1; k += 32) acc += partials[(uint64_t)k * n + i];
    acc = warp_sum_f64(acc);
    finite = finite && isfinite(acc);
    norms[i] = sqrt(acc);  // IEEE correctly rounded (np.linalg.norm = sqrt(dot))
    if (lane == 0) sumsq[(uint64_t)t * n + i] = acc;
  }
  if (lane != 0) return;
  int32_t st = finite ? 0 : 2;
  double target = 1.0;
  if (target_mode == 1) {  // fusion.py:95-99: mean of the non-zero norms (Python sum order)
    double sum = 0.0;
    int cnt = 0;
    for (int i = 0; i < n; ++i)
      if (norms[i] > 0.0) { sum = sum + norms[i]; ++cnt; }
    if (cnt == 0 && st == 0) st = 1;
    target = cnt ? sum / (double)cnt : 0.0;
  } else if (target_mode == 2) {
    target = target_value;
  }
  for (int i = 0; i < n; ++i) {
    // fusion.py:102: zero vectors pass through; otherwise delta * (target / norm)
    const double sc = (target_mode == 0 || norms[i] == 0.0) ? 1.0 : target / norms[i];
    scale[(uint64_t)t * n + i] = sc;
  }
  status[t] = st;
}

// ------------------------------------------------------------------ K2: dropout keep bitmap
// High word of mix64(z) (core.py:42-49) with the second product computed for its high word only:
// hi32(z * K2 mod 2^64) = hi32(lo * K2lo) + lo * K2hi + hi * K2lo (mod 2^32); the final
// z ^= z >> 31 changes the high word to h ^ (h >> 31).
// High word of z * kMix2 mod 2^64 after the first two SplitMix64 rounds (core.py:42-49):
// hi32(z * K2) = hi32(lo * K2lo) + lo * K2hi + hi * K2lo (mod 2^32).
__device__ __forceinline__ uint32_t mix64_pre_hi(uint64_t z) {
  z ^= z >> 30;
  z *= kMix1;
  z ^= z >> 27;
  const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
  return __umulhi(lo, (uint32_t)kMix2) + lo * (uint32_t)(kMix2 >> 32) + hi * (uint32_t)kMix2;
}

// bits = 2 * bits + (x >= y): one subtract-with-carry and one add-with-carry (no predicates, no SEL)
__device__ __forceinline__ uint32_t push_ge(uint32_t bits, uint32_t x, uint32_t y) {
  uint32_t r;
  asm("{\n .reg .u32 t;\n sub.cc.u32 t, %1, %2;\n addc.u32 %0, %3, %3;\n}" : "=r"(r) : "r"(x), "r"(y), "r"(bits));
  return r;
}
// bits = 2 * bits + (x >= y) for 64-bit x, y
__device__ __forceinline__ uint32_t push_ge64(uint32_t bits, uint64_t x, uint64_t y) {
  uint32_t r;
  asm("{\n .reg .u32 t;\n sub.cc.u32 t, %1, %3;\n subc.cc.u32 t, %2, %4;\n addc.u32 %0, %5, %5;\n}"
      : "=r"(r)
      : "r"((uint32_t)x), "r"((uint32_t)(x >> 32)), "r"((uint32_t)y), "r"((uint32_t)(y >> 32)), "r"(bits));
  return r;
}

// MODE 0: keep <=> mix64(c) >= t64 (full 64-bit draw).  MODE 1: t64 has a zero low word (e.g. p = 0.3
// rounded to 2^-32 steps), so the high word decides: h ^ (h >> 31) >= t_hi.  MODE 2: additionally t_hi
// is even (p = 0.5, 0.25, 0.75, ...): the final xor-shift only touches bit 0 of the high word, which
// cannot move it across an even threshold, so h >= t_hi.  All three are exact.  Bits are assembled
// from draw 31 down to draw 0 (add-with-carry doubling), so draw j lands in bit j.
template <int MODE>
__global__ void k_mask_bitmap(ulonglong4 seeds_lo, ulonglong4 seeds_hi, int n, uint64_t thresh, uint64_t w_lo,
                              uint64_t n_bits, uint32_t* __restrict__ bitmap, uint64_t words_per_row) {
  // keep iff (mix64(c_j) >> 11) >= thresh  <=>  mix64(c_j) >= thresh << 11  (thresh <= 2^53)
  const uint64_t t64 = thresh << 11;
  const uint32_t t_hi = (uint32_t)(t64 >> 32);
  const uint64_t words = (n_bits + 31) / 32;
  const int i = blockIdx.y;  // expert (grid.y = N): no 64-bit division per word
  const uint64_t seed = i < 4 ? (&seeds_lo.x)[i] : (&seeds_hi.x)[i - 4];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = w_lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words; w += stride) {
    uint32_t bits = 0;
    uint64_t c = seed + (w * 32 + 32) * kGamma;  // counter of draw j = 32 w + 31 (core.py:69-71)
#pragma unroll 8
    for (int b = 31; b >= 0; --b) {
      if (MODE == 2) {
        bits = push_ge(bits, mix64_pre_hi(c), t_hi);
      } else if (MODE == 1) {
        const uint32_t h = mix64_pre_hi(c);
        bits = push_ge(bits, h ^ (h >> 31), t_hi);
      } else {
        bits = push_ge64(bits, mix64(c), t64);
      }
      c -= kGamma;
    }
    bitmap[(uint64_t)i * words_per_row + w] = bits;
  }
}

// ------------------------------------------------------------------ K3: merge
struct MergeArgs {
  rlk_fusion_plan plan;
  const double* scale;  // [n_tensors * N]
  double w[RLK_MAX_EXPERTS];
  uint64_t seed[RLK_MAX_EXPERTS];
  uint64_t thresh;
  double keep_prob, inv_keep;
  uint64_t words_per_row;
  unsigned long long* counters;
  int dropout_mode, erase_mode, delta_mode, with_base, fast;
  uint32_t stage_bytes, nstages;
  const uint32_t* bitmap;
  uint32_t sub_shift;  // K3 work unit = 1 / 2^sub_shift of an item (small layouts: more CTAs busy)
  // deferred exact path of the bf16 fast merge: per CTA a queue of flagged elements (segment, element)
  // and its length, finished by k_merge_fixup after the merge (null: exact path inside the merge)
  uint4* fix_q;  // entries of kFixWords<N> uint4: segment | keep << 24, element, the bf16 inputs
  uint32_t* fix_count;
  uint32_t fix_cap;        // entries per CTA (set at launch from the total)
  uint64_t fix_cap_total;  // entries in the caller's workspace
};

struct ElemConsts {
  double scale[RLK_MAX_EXPERTS];
};

// uint4 words per fix-up queue entry: segment | keep << 24, element, then 1 + N bf16 inputs
template <int N> constexpr int kFixWords = N <= 3 ? 1 : 2;
static_assert(RLK_MAX_EXPERTS <= 8, "a fix-up entry holds at most 9 bf16 inputs and 8 keep bits");

// RN(a / b) from r = RN(1/b): q = RN(a r); e = a - q b (exact by FMA); RN(q + e r) (Markstein).
__device__ __forceinline__ double div_rn(double a, double b, double r) {
  const double q = __dmul_rn(a, r);
  const double e = fma(-q, b, a);
  return fma(e, r, q);
}

// Reference-order f64 evaluation of one element (exact semantics of fusion.py:102, 114, 130-141, 184-186).
// keep: bit i = dropout keep decision of expert i.  Returns fused value; nz/er: bit i set when
// expert i's entry is non-zero after dropout / was erased.
template <int N>
__device__ __forceinline__ double merge_elem_f64(double B, const double* X, uint32_t keep, const MergeArgs& a,
                                                 const ElemConsts& c, uint32_t& nz, uint32_t& er) {
  double K[N];
  nz = 0;
  er = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double D = a.delta_mode ? X[i] : __dsub_rn(X[i], B);
    double k = __dmul_rn(D, c.scale[i]);
    if (a.dropout_mode) k = ((keep >> i) & 1u) ? div_rn(k, a.keep_prob, a.inv_keep) : 0.0;
    K[i] = k;
    nz |= (uint32_t)(k != 0.0) << i;
  }
  if (N >= 2 && a.erase_mode) {
    double V;
    if (a.erase_mode == 1) {
      V = K[0];
#pragma unroll
      for (int i = 1; i < N; ++i) V = __dadd_rn(V, K[i]);
    } else {
      auto sq = [](double k) {
        const double s = k > 0.0 ? 1.0 : (k < 0.0 ? -1.0 : (k == 0.0 ? 0.0 : k));
        return __dmul_rn(s, __dmul_rn(k, k));
      };
      V = sq(K[0]);
#pragma unroll
      for (int i = 1; i < N; ++i) V = __dadd_rn(V, sq(K[i]));
    }
    const int maj = V > 0.0 ? 1 : (V < 0.0 ? -1 : 0);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const bool opp = (maj > 0 && K[i] < 0.0) || (maj < 0 && K[i] > 0.0);
      if (opp) {
        K[i] = 0.0;
        er |= 1u << i;
      }
    }
  }
  double Y = B;
#pragma unroll
  for (int i = 0; i < N; ++i) Y = __dadd_rn(Y, __dmul_rn(a.w[i], K[i]));
  return Y;
}

// The same reference-order f64 evaluation with the dropout / erase modes fixed at compile time (DROP 0
// none, 2 bitmap; ERASE 0 off, 1 sum, 2 squared) for base + experts in pair mode.  s[i] is the
// normalisation scale, or with FOLD the scale times 1/keep_prob: when 1/keep_prob is a power of two
// and s[i] >= 2^-873, RN(RN(d s) / keep_prob) == RN(d (s / keep_prob)) for every difference d of two
// f32 values (|d| >= 2^-149 when non-zero, so d s never underflows), saving the Markstein division.
template <int N, int DROP, int ERASE, bool FOLD>
__device__ __forceinline__ double merge_elem_spec(double B, const double* X, uint32_t keep, const MergeArgs& a,
                                                  const double* s, uint32_t& er) {
  double K[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double k = __dmul_rn(__dsub_rn(X[i], B), s[i]);
    if constexpr (DROP != 0) {
      if constexpr (!FOLD) k = div_rn(k, a.keep_prob, a.inv_keep);
      k = ((keep >> i) & 1u) ? k : 0.0;
    }
    K[i] = k;
  }
  er = 0;
  if constexpr (N >= 2 && ERASE != 0) {
    double V;
    if constexpr (ERASE == 1) {
      V = K[0];
#pragma unroll
      for (int i = 1; i < N; ++i) V = __dadd_rn(V, K[i]);
    } else {
      auto sq = [](double k) {
        const double m = __dmul_rn(k, k);
        return k > 0.0 ? m : (k < 0.0 ? -m : __dmul_rn(k, m));  // sign(k) * k^2 (sign(0) = 0, NaN stays NaN)
      };
      V = sq(K[0]);
#pragma unroll
      for (int i = 1; i < N; ++i) V = __dadd_rn(V, sq(K[i]));
    }
    const bool vp = V > 0.0, vn = V < 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const bool opp = (vp & (K[i] < 0.0)) | (vn & (K[i] > 0.0));  // no short-circuit branches
      K[i] = opp ? 0.0 : K[i];
      er |= (uint32_t)opp << i;
    }
  }
  double Y = B;
#pragma unroll
  for (int i = 0; i < N; ++i) Y = __dadd_rn(Y, __dmul_rn(a.w[i], K[i]));
  return Y;
}

// One ring stage of the specialised f32 merge: VEC = 4 elements per 16-byte vector, the keep bits of a
// vector read as one 4-bit field per expert.
template <int N, int DROP, int ERASE, bool FOLD>
__device__ __forceinline__ void merge_stage_f32(const uint8_t* sb, const uint8_t* bm, uint32_t nvec, int tid,
                                                const MergeArgs& a, const double* s, void* out, uint64_t out_base,
                                                uint32_t* cnt_er) {
  constexpr uint32_t SB = StreamBytes<N>::v;
  constexpr uint32_t BMW = SB / 4 / 32;  // bitmap words per expert per stage
  for (uint32_t v = tid; v < nvec; v += kCThreads) {
    const uint32_t le = v * 4;
    double b[4], x[N][4];
    VecIO<RLK_F32>::f64(lds128(sb + v * 16), b);
#pragma unroll
    for (int i = 0; i < N; ++i) VecIO<RLK_F32>::f64(lds128(sb + (i + 1) * SB + v * 16), x[i]);
    uint32_t kb[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      kb[i] = 0xfu;
      if constexpr (DROP != 0) kb[i] = reinterpret_cast<const uint32_t*>(bm)[i * BMW + (le >> 5)] >> (le & 31);
    }
    double y[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      double X[N];
      uint32_t keep = 0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        X[i] = x[i][e];
        keep |= ((kb[i] >> e) & 1u) << i;
      }
      uint32_t erm;
      y[e] = merge_elem_spec<N, DROP, ERASE, FOLD>(b[e], X, keep, a, s, erm);
#pragma unroll
      for (int i = 0; i < N; ++i) cnt_er[i] += (erm >> i) & 1u;
    }
    store_vec_f64<RLK_F32, 4>(out, out_base + le, y);
  }
}

template <int N, int VEC>
__device__ __forceinline__ uint32_t keep_bits_for(const MergeArgs& a, const uint8_t* bm_stage, uint32_t bm_stride,
                                                  uint32_t local_elem, uint64_t jglobal, int e) {
  // returns N-bit keep mask for element local_elem + e
  uint32_t m = 0;
  if (a.dropout_mode == 0) return (1u << N) - 1u;
  if (a.dropout_mode == 2) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const uint32_t word = reinterpret_cast<const uint32_t*>(bm_stage + i * bm_stride)[(local_elem + e) >> 5];
      m |= ((word >> ((local_elem + e) & 31)) & 1u) << i;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) m |= (uint32_t)keep_draw(a.seed[i], jglobal + e, a.thresh) << i;
  }
  return m;
}

// Out-of-line exact evaluation used by the fast path for the rare elements whose guard tripped
// (one copy of the f64 code instead of one per unrolled element).
template <int N>
struct FArr { float v[N]; };

template <int N>
__device__ __noinline__ double merge_elem_slow(float b, FArr<N> x, uint32_t keep, const MergeArgs* a,
                                              const double* scale, uint32_t* nz, uint32_t* er) {
  ElemConsts c;
  double X[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    c.scale[i] = scale[i];
    X[i] = (double)x.v[i];
  }
  return merge_elem_f64<N>((double)b, X, keep, *a, c, *nz, *er);
}

// Fast-path erase decisions of one element, recomputed with exactly the phase-1 arithmetic (scalar
// IEEE ops give the same bits as the packed f32x2 ones); used to replace the counts of slow elements.
template <int N>
__device__ __forceinline__ uint32_t fast_opp_bits(float b, const float* x, uint32_t keep, const float* sr32,
                                                  int erase_mode, bool delta) {
  float k[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const float d = delta ? x[i] : fmaf(b, -1.f, x[i]);
    k[i] = __fmul_rn(d, ((keep >> i) & 1u) ? sr32[i] : 0.f);
  }
  // the same operations as the packed phase 1: sum mode adds, squared mode k0|k0| then fused k_i|k_i| + v
  float v = erase_mode == 1 ? k[0] : __fmul_rn(k[0], fabsf(k[0]));
#pragma unroll
  for (int i = 1; i < N; ++i) v = erase_mode == 1 ? __fadd_rn(v, k[i]) : __fmaf_rn(k[i], fabsf(k[i]), v);
  const float sg = copysignf(1.f, v);
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) m |= (uint32_t)(__fmul_rn(k[i], sg) < 0.f) << i;
  return m;
}

// Phase-2 resolver: one flagged element re-evaluated in scalar f32 (exact ties, and elements flagged by
// a margin the scalar re-check can still certify).  ERASE 0 / 1 only (the squared vote keeps the f64 path).  Returns
//   1: certified like the fast path (same vote-sign and output-bracket arguments); the fast loop's
//      erased count for this element stands;
//   2: an exact sum-vote tie, certified: with every scale an exact power of two and no dropout or a
//      power-of-two keep probability (`tie_ok`), k_i = d_i * sr is exact in f32 when the non-zero
//      members of {b, kept x_i} span at most 13 binades (d_i then needs <= 22 bits), and so are the
//      vote's partial sums (< 2^24 quanta); the reference's f64 k_i and vote are exact too.  A vote
//      computed as exactly 0 is then a true tie (fusion.py:136-141: sign(0) = 0 erases nothing), and
//      `fast_opp` is what the fast loop counted as erased (t = k * sign(+0) < 0), to be undone;
//   0: not certifiable here -- the caller runs the reference-order f64 path.
// sr32 / w32 / wh32 / wmax are the kernel's scaled-domain constants (k' = k 2^24, w' = w 2^-24).
template <int N, int ERASE, bool UNI>
__device__ __forceinline__ int scalar_resolve(uint32_t bbits, const uint32_t* xbits, uint32_t keep, const float* sr32,
                                              const float* w32, const float* wh32, float wmax, bool tie_ok,
                                              uint16_t* out, uint32_t* fast_opp) {
  const float be = __uint_as_float(bbits << 16);
  float k[N];
#pragma unroll
  for (int i = 0; i < N; ++i)
    k[i] = __fmul_rn(fmaf(be, -1.f, __uint_as_float(xbits[i] << 16)), ((keep >> i) & 1u) ? sr32[i] : 0.f);
  float aa = N == 1 ? fabsf(k[0]) : __fadd_rn(fabsf(k[0]), fabsf(k[1]));
#pragma unroll
  for (int i = 2; i < N; ++i) aa = __fadd_rn(aa, fabsf(k[i]));
  const float S = fmaf(wmax, aa, __fadd_rn(fabsf(be), 0x1p-110f));
  float y;
  int kind = 1;
  if constexpr (ERASE == 1 && N >= 2) {
    float vv = k[0];
#pragma unroll
    for (int i = 1; i < N; ++i) vv = __fadd_rn(vv, k[i]);
    if (fmaf(-0x1p-20f, aa, fabsf(vv)) < 0.f || !(aa < INFINITY)) {  // vote sign not certain here
      if (!(tie_ok && vv == 0.f)) return 0;
      uint32_t emax = 0, emin = 0xffu;
      auto span = [&](uint32_t h) {
        if (h & 0x7fffu) {
          const uint32_t e = max((h >> 7) & 0xffu, 1u);  // subnormals: the ulp of binade 1
          emax = max(emax, e);
          emin = min(emin, e);
        }
      };
      span(bbits);
#pragma unroll
      for (int i = 0; i < N; ++i)
        if ((keep >> i) & 1u) span(xbits[i]);
      if (emax < emin || emax - emin > 13u) return 0;
      // a true tie: nothing erased, y = b + sum_i w_i k_i
      y = be;
      uint32_t fo = 0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        y = fmaf(w32[i], k[i], y);
        fo |= (uint32_t)(k[i] < 0.f) << i;
      }
      *fast_opp = fo;
      kind = 2;
    } else {
      const float sg = copysignf(1.f, vv);
      if constexpr (UNI) {
        y = fmaf(wh32[0], fmaf(sg, aa, vv), be);
      } else {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const float t = fmaf(k[i], sg, 0.f);
          acc = fmaf(wh32[i], __fadd_rn(t, fabsf(t)), acc);
        }
        y = fmaf(sg, acc, be);
      }
    }
  } else {
    y = be;
#pragma unroll
    for (int i = 0; i < N; ++i) y = fmaf(w32[i], k[i], y);
  }
  if (!(fabsf(y) < INFINITY)) return 0;
  constexpr float kBr = (float)(N + 7) * 0x1p-24f;  // the fast path's bracket (its error bound covers both kinds)
  const uint16_t lo = f32_to_bf16_rne(fmaf(-kBr, S, y)), hi = f32_to_bf16_rne(fmaf(kBr, S, y));
  if (lo != hi) return 0;
  *out = lo;
  return kind;
}

__device__ __forceinline__ uint32_t word_of(const uint4& q, int p) {
  return p == 0 ? q.x : (p == 1 ? q.y : (p == 2 ? q.z : q.w));
}

// Generic K3: the reference-order f64 path for every dtype combination (and the tails).
// SPEC != 0 (f32 -> f32 pair mode, 2..4 experts): the modes are compile-time, SPEC = 1 + 3 * (DROP / 2) + ERASE.
template <int DTI, int DTO, int N, int SPEC = 0>
__global__ void __launch_bounds__(kThreads, N <= 5 ? 2 : 1) k_merge(const __grid_constant__ MergeArgs a) {
  static_assert(SPEC == 0 || (DTI == RLK_F32 && DTO == RLK_F32 && N >= 2 && N <= 4), "specialised merge: f32 only");
  constexpr int SDROP = SPEC ? 2 * ((SPEC - 1) / 3) : 0;
  constexpr int SERASE = SPEC ? (SPEC - 1) % 3 : 0;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int ESZ = Elem<DTI>::size;
  constexpr int VEC = 16 / ESZ;
  constexpr uint32_t SB = StreamBytes<N>::v;
  constexpr uint32_t ELEMS = SB / ESZ;
  constexpr uint32_t BMB = ELEMS / 8;
  const Ring r = ring_setup(smem, a.stage_bytes, a.nstages);
  const bool delta = a.delta_mode != 0;
  const bool wb = a.with_base != 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == kCWarps) {
    if (lane == 0)
      produce<ESZ, N>(a.plan, r, wb, a.dropout_mode == 2 ? a.bitmap : nullptr, a.words_per_row, a.sub_shift);
    return;
  }
  const int tid = threadIdx.x;
  RingPos q;
  SegCursor cur;
  const uint32_t unit = kItem >> a.sub_shift;
  for (uint32_t u = blockIdx.x; u < (a.plan.n_items << a.sub_shift); u += gridDim.x) {
    const uint32_t item = u >> a.sub_shift;
    const ItemGeom g = item_geom(a.plan, cur, item);
    const uint32_t lo = (u & ((1u << a.sub_shift) - 1u)) * unit;
    if (lo >= g.len) continue;
    const uint32_t hi = min(g.len, lo + unit);
    const double* scale = a.scale + (uint64_t)g.tensor * N;
    ElemConsts c;
#pragma unroll
    for (int i = 0; i < N; ++i) c.scale[i] = __ldg(scale + i);
    // specialised path: fold 1/keep_prob into the scale when that is exact (see merge_elem_spec)
    bool fold = false;
    double sf[N];
    if constexpr (SPEC != 0) {
      fold = SDROP != 0 && (__double_as_longlong(a.inv_keep) & 0x000fffffffffffffull) == 0 &&
             __dmul_rn(a.inv_keep, a.keep_prob) == 1.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        sf[i] = __dmul_rn(c.scale[i], a.inv_keep);
        fold = fold && (c.scale[i] == 0.0 || c.scale[i] >= 0x1p-873) && fabs(sf[i]) < INFINITY;
      }
#pragma unroll
      for (int i = 0; i < N; ++i) sf[i] = fold ? sf[i] : c.scale[i];
    }
    uint32_t cnt_er[N];  // entries erased (non-zero entries after dropout are counted by K1)
#pragma unroll
    for (int i = 0; i < N; ++i) cnt_er[i] = 0;
    const uint64_t jtensor0 = g.j0 + g.start;
    for (uint32_t off = lo; off < hi; off += ELEMS) {
      const uint32_t n = min(ELEMS, hi - off);
      const uint32_t main_elems = ((n * ESZ) & ~15u) / ESZ;
      const uint32_t s = q.s, ph = q.ph;
      mbar_wait(&r.full[s], ph);
      const uint8_t* sb = r.buf + s * r.stage_bytes;
      const uint8_t* bm = sb + (N + 1) * SB;
      const uint32_t nvec = main_elems / VEC;
      const uint64_t out_base = g.start + off;
      if constexpr (SPEC != 0) {
        if (fold) merge_stage_f32<N, SDROP, SERASE, true>(sb, bm, nvec, tid, a, sf, g.out, out_base, cnt_er);
        else merge_stage_f32<N, SDROP, SERASE, false>(sb, bm, nvec, tid, a, sf, g.out, out_base, cnt_er);
      } else {
        // ---------------- reference-order f64 path
        for (uint32_t v = tid; v < nvec; v += kCThreads) {
          const uint32_t le = v * VEC;
          double b[VEC], x[N][VEC];
          if (wb) VecIO<DTI>::f64(lds128(sb + v * 16), b);
          else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) b[e] = 0.0;
          }
#pragma unroll
          for (int i = 0; i < N; ++i) VecIO<DTI>::f64(lds128(sb + (i + (wb ? 1 : 0)) * SB + v * 16), x[i]);
          double y[VEC];
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            double X[N];
#pragma unroll
            for (int i = 0; i < N; ++i) X[i] = x[i][e];
            const uint32_t keep = keep_bits_for<N, VEC>(a, bm, BMB, le, jtensor0 + off + le, e);
            uint32_t nzm, erm;
            y[e] = merge_elem_f64<N>(b[e], X, keep, a, c, nzm, erm);
#pragma unroll
            for (int i = 0; i < N; ++i) cnt_er[i] += (erm >> i) & 1u;
          }
          store_vec_f64<DTO, VEC>(g.out, out_base + le, y);
        }
      }
      // tail elements (fewer than 16 bytes) straight from global memory
      for (uint32_t e = main_elems + tid; e < n; e += kCThreads) {
        const uint64_t idx = g.start + off + e;
        const double B = wb ? load_f64<DTI>(g.seg->base, idx) : 0.0;
        double X[N];
#pragma unroll
        for (int i = 0; i < N; ++i) X[i] = load_f64<DTI>(g.seg->expert[i], idx);
        uint32_t keep = (1u << N) - 1u;
        if (a.dropout_mode) {
          keep = 0;
#pragma unroll
          for (int i = 0; i < N; ++i) keep |= (uint32_t)keep_draw(a.seed[i], jtensor0 + off + e, a.thresh) << i;
        }
        uint32_t nzm, erm;
        const double Y = merge_elem_f64<N>(B, X, keep, a, c, nzm, erm);
#pragma unroll
        for (int i = 0; i < N; ++i) cnt_er[i] += (erm >> i) & 1u;
        (void)nzm;
        store_from_f64<DTO>(g.out, idx, Y);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&r.empty[s]);
      q.next(r.nstages);
    }
    // per-item counters -> per-tensor u64 totals (integer atomics: order-independent)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const uint32_t er = __reduce_add_sync(0xffffffffu, cnt_er[i]);
      if (lane == 0 && er) atomicAdd(a.counters + (uint64_t)g.tensor * 2 * N + N + i, (unsigned long long)er);
    }
  }
}


__device__ __forceinline__ uint32_t mask_ne0(float x) {  // 0xffffffff iff x != 0
  uint32_t r;
  asm("set.ne.u32.f32 %0, %1, 0f00000000;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ uint32_t mask_lt0(float x) {  // 0xffffffff iff x < 0 (false for -0)
  uint32_t r;
  asm("set.lt.u32.f32 %0, %1, 0f00000000;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float andnot_f(float x, uint32_t m) { return __uint_as_float(__float_as_uint(x) & ~m); }
// c + (x >> 31): hi32(x * 2) + c (mad.hi; ptxas emits it as one LEA.HI)
__device__ __forceinline__ uint32_t add_sign_bit(uint32_t x, uint32_t c) {
  uint32_t r;
  asm("mad.hi.u32 %0, %1, 2, %2;" : "=r"(r) : "r"(x), "r"(c));
  return r;
}
// PRMT in sign-replicate mode: each result byte = 0x00 / 0xFF from the sign bit of the selected byte
__device__ __forceinline__ uint32_t prmt_sign(uint32_t x, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(x), "r"(sel));
  return r;
}
// (x & m) | (b & ~m) in one LOP3
__device__ __forceinline__ uint32_t select_halves(uint32_t x, uint32_t b, uint32_t m) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xe4;" : "=r"(r) : "r"(x), "r"(b), "r"(m));
  return r;
}
// (lo, hi) bf16 halves of w minus the f32 pair b, each rounded once to f32 (sub.rn.f32.bf16: one
// FHADD.BF16 per element reading the bf16 half in place -- no unpacking)
__device__ __forceinline__ float2 bf16x2_minus_f32(uint32_t w, float2 b) {
  float2 r;
  asm("{\n .reg .b16 lo, hi;\n mov.b32 {lo, hi}, %2;\n sub.rn.f32.bf16 %0, lo, %3;\n sub.rn.f32.bf16 %1, hi, %4;\n}"
      : "=f"(r.x), "=f"(r.y)
      : "r"(w), "f"(b.x), "f"(b.y));
  return r;
}
// min that propagates NaN (min.NaN.f32): a NaN guard margin must force the exact path
__device__ __forceinline__ float fmin_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fmin3_nan(float a, float b, float c) {
  float r;
  asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// +-1.0f with the sign of x (one LOP3)
__device__ __forceinline__ float sign_one(float x) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xea;" : "=r"(r) : "r"(__float_as_uint(x)), "r"(0x80000000u), "r"(0x3f800000u));
  return __uint_as_float(r);
}
// (x, y) rounded to nearest-even bf16, packed lo | hi << 16 (one F2FP)
__device__ __forceinline__ uint32_t pack_bf16x2(float2 v) {
  __nv_bfloat162 p = __floats2bfloat162_rn(v.x, v.y);
  return *reinterpret_cast<uint32_t*>(&p);
}

// Fast K3 for bf16 experts + bf16 base -> bf16 (the checkpoint path): f32x2 arithmetic with certified
// guards; DROP 0 = no dropout, 2 = keep bits from the K2 bitmap; ERASE 0 off, 1 sum vote, 2 squared vote.
// Elements whose guard trips are recomputed exactly (merge_elem_slow) in a rarely-taken phase 2.
// Per-thread unit of the fast merge: kFastElems bf16 elements (kFastPairs 32-bit words) per stream.
#ifndef RLK_FAST_PAIRS
#define RLK_FAST_PAIRS 2
#endif
constexpr int kFastPairs = RLK_FAST_PAIRS;
#ifndef RLK_FAST_SB
#define RLK_FAST_SB 16384
#endif
constexpr uint32_t kFastSB = RLK_FAST_SB;  // bytes per stream per stage in the fast merge
constexpr int kFastElems = 2 * kFastPairs;
#ifndef RLK_FAST_CTAS
#define RLK_FAST_CTAS 1
#endif
constexpr int kFastCtas = RLK_FAST_CTAS;  // CTAs per SM of the fast merge (the smem budget is split)
struct FastVec {
  uint32_t w[kFastPairs];
  __device__ static FastVec load(const void* p) {
    FastVec v;
    if constexpr (kFastPairs == 4) {
      const uint4 q = lds128(p);
      v.w[0] = q.x; v.w[1] = q.y; v.w[2] = q.z; v.w[3] = q.w;
    } else if constexpr (kFastPairs == 2) {
      uint2 q;
      asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(q.x), "=r"(q.y) : "r"(smem_u32(p)));
      v.w[0] = q.x; v.w[1] = q.y;
    } else {
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v.w[0]) : "r"(smem_u32(p)));
    }
    return v;
  }
  __device__ static void store(void* p, const uint32_t* w) {
    if constexpr (kFastPairs == 4) {
      stg128_stream(p, make_uint4(w[0], w[1], w[2], w[3]));
    } else if constexpr (kFastPairs == 2) {
      asm volatile("st.global.L1::no_allocate.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(w[0]), "r"(w[1]) : "memory");
    } else {
      asm volatile("st.global.L1::no_allocate.u32 [%0], %1;" ::"l"(p), "r"(w[0]) : "memory");
    }
  }
};

template <int N, int DROP, int ERASE, bool UNI>
__global__ void __launch_bounds__(kFastThreads, kFastCtas) k_merge_fast(const __grid_constant__ MergeArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr uint32_t SB = kFastSB;
  constexpr uint32_t ELEMS = SB / 2;
  constexpr uint32_t BMB = ELEMS / 8;
  constexpr bool kErase = (ERASE != 0) && (N >= 2);
  __shared__ uint32_t fix_n;  // flagged elements this CTA queued for k_merge_fixup
#ifdef RLK_DEBUG_FLAGS
  uint32_t dbg_vote = 0, dbg_brk = 0;
#endif
  if (threadIdx.x == 0) fix_n = 0;
  const Ring r = ring_setup(smem, a.stage_bytes, a.nstages, kFastCWarps);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == kFastCWarps) {
    if (lane == 0) produce<2, N, kFastSB>(a.plan, r, true, DROP == 2 ? a.bitmap : nullptr, a.words_per_row, a.sub_shift);
    return;
  }
  const int tid = threadIdx.x;
  // 4 elements per thread: the thread's keep bits are the low (even tid) or high (odd tid) nibble of a
  // bitmap byte, every iteration (le & 4 == (tid & 1) * 4 since kFastCThreads is even).  Multiplying
  // the masked nibble moves bit k to bit 8k + 7 (distinct partial products, no carries).
  const uint32_t nib_mask = (tid & 1) ? 0xf0u : 0x0fu;
  const uint32_t nib_mul = (tid & 1) ? 0x01020408u : 0x10204080u;
  const float cv = ERASE == 1 ? 0x1p-20f : 0x1p-19f;
  constexpr float kBr = (float)(N + 7) * 0x1p-24f;  // output bracket half-width / S (see the bound below)
  // Scaled domain (ERASE 0 / 1): the kernel works with k' = k * 2^24 and folds 2^-24 into the weights
  // (both exact power-of-two scalings).  Every non-zero k' is then a normal float (|d| >= 2^-133,
  // sr >= 2^-16), so its rounding error is relative, and the vote's partial sums are either normal or
  // subnormal-and-exact: the vote's relative error bound needs no subnormal guard.  What can still be
  // tiny are the weighted terms of y, covered by the 2^-110 floor in S below.  The squared vote
  // (ERASE 2) would square the scale: it keeps k unscaled and its own floor check.
  constexpr float kKS = ERASE == 2 ? 1.f : 0x1p24f;
  constexpr float kKSinv = ERASE == 2 ? 1.f : 0x1p-24f;
  float w32[N], wh32[N];
  float wmax = 0.f;
  bool w_ok = true;  // w * 2^-24 exact and normal: every weight zero or >= 2^-100
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const float w = (float)a.w[i];
    w_ok = w_ok && (w == 0.f || w >= 0x1p-100f);
    w32[i] = w * kKSinv;
    wh32[i] = 0.5f * w32[i];
    wmax = fmaxf(wmax, w32[i]);
  }
  RingPos q;
  SegCursor cur;
  ElemConsts c;
  float sr32[N];
  bool fast_ok = false, tie_ok = false;
  uint32_t c_tensor = 0xffffffffu;  // tensor whose scales are loaded
  // exact ties need power-of-two keep scaling (checked on the f64 value the reference divides by)
  const bool keep_pow2 = !DROP || (__double_as_longlong(a.keep_prob) & 0xfffffffffffffull) == 0;
  const uint32_t unit = kItem >> a.sub_shift;
  for (uint32_t u = blockIdx.x; u < (a.plan.n_items << a.sub_shift); u += gridDim.x) {
    const uint32_t item = u >> a.sub_shift;
    const ItemGeom g = item_geom(a.plan, cur, item);
    const uint32_t lo = (u & ((1u << a.sub_shift) - 1u)) * unit;
    if (lo >= g.len) continue;
    const uint32_t hi = min(g.len, lo + unit);
    const double* scale = a.scale + (uint64_t)g.tensor * N;
    uint16_t* const outp = (uint16_t*)g.out;
    if (g.tensor != c_tensor) {  // per-tensor constants: reloaded only when the tensor changes
      c_tensor = g.tensor;
      fast_ok = w_ok;
      tie_ok = ERASE == 1 && keep_pow2;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        c.scale[i] = __ldg(scale + i);
        sr32[i] = (float)(DROP ? c.scale[i] / a.keep_prob : c.scale[i]);
        // k = d * sr cannot underflow for bf16 deltas (|d| >= 2^-133) when sr >= 2^-16; sr < 2^100
        // keeps sr * 2^24 finite
        fast_ok = fast_ok && sr32[i] >= 0x1p-16f && sr32[i] < 0x1p100f;
        // tie resolution: every scale an exact power of two (f64 mantissa zero), hence all sr exact
        tie_ok = tie_ok && (__double_as_longlong(c.scale[i]) & 0xfffffffffffffull) == 0 && c.scale[i] > 0.0;
        sr32[i] *= kKS;
      }
    }
    uint32_t cnt_er[N];  // entries erased (non-zero entries after dropout are counted by K1)
#pragma unroll
    for (int i = 0; i < N; ++i) cnt_er[i] = 0;
    const uint64_t jtensor0 = g.j0 + g.start;
    for (uint32_t off = lo; off < hi; off += ELEMS) {
      const uint32_t n = min(ELEMS, hi - off);
      const uint32_t main_elems = ((n * 2) & ~15u) / 2;
      const uint32_t s = q.s, ph = q.ph;
      mbar_wait(&r.full[s], ph);
      const uint8_t* sb = r.buf + s * r.stage_bytes;
      const uint8_t* bm = sb + (N + 1) * SB;
      const uint32_t nvec = main_elems / kFastElems;
      const uint64_t out_base = g.start + off;
      // elements whose guard trips are only recorded here (bit kFastElems * j + e: iteration j, element
      // e) and recomputed after the stage's fast loop, so the hot loop carries no slow-path code and a
      // warp pays max-over-lanes(popcount) slow rounds per stage, not one per element position
      static_assert(ELEMS / kFastElems / kFastCThreads * kFastElems <= 32, "slow bits per stage exceed a word");
      uint32_t slowbits = 0;
      auto vec = [&](const uint32_t v, const uint32_t jit) {
        const uint32_t le = v * kFastElems;
        RLK_DCHECK(le + kFastElems <= main_elems && jit + kFastElems <= 32);
        const FastVec bw4 = FastVec::load(sb + v * (2 * kFastElems));
        FastVec xw4[N];
        uint32_t kb[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          xw4[i] = FastVec::load(sb + (i + 1) * SB + v * (2 * kFastElems));
          kb[i] = DROP ? (uint32_t)bm[i * BMB + (le >> 3)] : 0xffu;
        }
        // dropout on the integer side: 4 keep bits at a time go to the sign bits of 4 bytes (one IMAD by
        // a per-thread multiplier that also picks the byte's low or high nibble; the other bits of the
        // product are ignored), PRMT sign-replication turns them into halfword masks, and one LOP3 per
        // word swaps every dropped expert half for the base half, so d = x - b is exactly +0 there
        // (reference: k = 0, fusion.py:114)
        static_assert(N <= 8, "the output bracket constant is derived for N <= 8 (RLK_MAX_EXPERTS)");
        uint32_t spread[N][(kFastElems + 3) / 4];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          if constexpr (kFastElems == 8) {
            spread[i][0] = DROP ? (kb[i] & 0x0fu) * 0x10204080u : 0u;
            spread[i][1] = DROP ? (kb[i] & 0xf0u) * 0x01020408u : 0u;
          } else {
            spread[i][0] = DROP ? (kb[i] & nib_mask) * nib_mul : 0u;
          }
        }
        uint32_t outw[kFastPairs];
        uint32_t mx[kFastPairs];  // bf16x2(y - margin) ^ bf16x2(y + margin): non-zero half -> recompute
        float2 gm[kFastPairs];    // vote / overflow margin per element: < 0 (or NaN) -> recompute it
#pragma unroll
        for (int p = 0; p < kFastPairs; ++p) {
          const uint32_t bw = bw4.w[p];
          const float2 b2 = make_float2(bf16_lo(bw), bf16_hi(bw));
          float2 k2[N];
#pragma unroll
          for (int i = 0; i < N; ++i) {
            uint32_t xw = xw4[i].w[p];
            if (DROP) xw = select_halves(xw, bw, prmt_sign(spread[i][p >> 1], (p & 1) ? 0xBBAAu : 0x9988u));
            const float2 d2 = bf16x2_minus_f32(xw, b2);
            k2[i] = __fmul2_rn(d2, make_float2(sr32[i], sr32[i]));
          }
          // sum |k| (|k0| + |k1| first: the abs modifiers ride on one FADD2, no add of zero)
          float2 aa;
          if constexpr (N == 1) {
            aa = make_float2(fabsf(k2[0].x), fabsf(k2[0].y));
          } else {
            aa = __fadd2_rn(make_float2(fabsf(k2[0].x), fabsf(k2[0].y)), make_float2(fabsf(k2[1].x), fabsf(k2[1].y)));
#pragma unroll
            for (int i = 2; i < N; ++i) aa = __fadd2_rn(aa, make_float2(fabsf(k2[i].x), fabsf(k2[i].y)));
          }
          // S = |b| + max w * sum|k| (+ 2^-110 in the scaled domain): a subnormal weighted term of y adds
          // at most 2^-150 absolute per rounding (N + 2 of them), which the floor covers with room to
          // spare (2^-20 S >= 2^-130 in the output bracket).  Overflow makes S infinite.
          float2 babs = make_float2(fabsf(b2.x), fabsf(b2.y));
          if constexpr (ERASE != 2) babs = __fadd2_rn(babs, make_float2(0x1p-110f, 0x1p-110f));
          const float2 S2 = __ffma2_rn(make_float2(wmax, wmax), aa, babs);
          float2 y2, g1;
          if constexpr (kErase) {
            float2 vv;
            if (ERASE == 1) {
              vv = k2[0];
#pragma unroll
              for (int i = 1; i < N; ++i) vv = __fadd2_rn(vv, k2[i]);
              // |vote| - 2^-20 sum|k'| (one rounding: its sign is exact).  < 0: the f32 vote's sign is not
              // certain (its error is <= 6 * 2^-24 sum|k'|, all of it relative: no subnormals in the
              // scaled domain); NaN: an overflow.  An all-zero column gives 0 - 0 = 0: an exact tie.
              g1 = __ffma2_rn(make_float2(-cv, -cv), aa, make_float2(fabsf(vv.x), fabsf(vv.y)));
            } else {
              // squared vote: sum k |k| against sum k^2 (error <= 11 * 2^-24 sum k^2 while k^2 is normal:
              // the floor check below)
              vv = __fmul2_rn(k2[0], make_float2(fabsf(k2[0].x), fabsf(k2[0].y)));
              float2 gg = __fmul2_rn(k2[0], k2[0]);
#pragma unroll
              for (int i = 1; i < N; ++i) {
                vv = __ffma2_rn(k2[i], make_float2(fabsf(k2[i].x), fabsf(k2[i].y)), vv);
                gg = __ffma2_rn(k2[i], k2[i], gg);
              }
              g1 = __ffma2_rn(make_float2(-cv, -cv), gg, make_float2(fabsf(vv.x), fabsf(vv.y)));
            }
            const float2 sg = make_float2(sign_one(vv.x), sign_one(vv.y));
            // t = k * sign(vote) + 0 (exact; +0 for k = 0): t < 0 <=> entry opposes the majority.
            // Erased entries are counted from t's sign bit; survivors enter as
            // w * max(t, 0) == (w / 2) * (t + |t|) exactly (both steps are power-of-two scalings)
            if constexpr (UNI) {
              // uniform weights w: sum_i w max(sg k_i, 0) = (w / 2) (sum_i k_i + sg sum_i |k_i|), so
              // y = b + (w / 2) (sum k + sg sum|k|); error <= (4 + 2 (N - 1) + 1) 2^-24 (|b| + w sum|k|)
              float2 vplain = k2[0];
#pragma unroll
              for (int i = 1; i < N; ++i) vplain = (ERASE == 1) ? vv : __fadd2_rn(vplain, k2[i]);
#pragma unroll
              for (int i = 0; i < N; ++i) {
                const float2 t2 = __ffma2_rn(k2[i], sg, make_float2(0.f, 0.f));
                cnt_er[i] = add_sign_bit(__float_as_uint(t2.x), cnt_er[i]);
                cnt_er[i] = add_sign_bit(__float_as_uint(t2.y), cnt_er[i]);
              }
              y2 = __ffma2_rn(make_float2(wh32[0], wh32[0]), __ffma2_rn(sg, aa, vplain), b2);
            } else {
              float2 acc = make_float2(0.f, 0.f);
#pragma unroll
              for (int i = 0; i < N; ++i) {
                const float2 t2 = __ffma2_rn(k2[i], sg, make_float2(0.f, 0.f));
                cnt_er[i] = add_sign_bit(__float_as_uint(t2.x), cnt_er[i]);
                cnt_er[i] = add_sign_bit(__float_as_uint(t2.y), cnt_er[i]);
                const float2 tp = __fadd2_rn(t2, make_float2(fabsf(t2.x), fabsf(t2.y)));
                acc = __ffma2_rn(make_float2(wh32[i], wh32[i]), tp, acc);
              }
              y2 = __ffma2_rn(sg, acc, b2);
            }
            // a finite vote and sum|k| do not rule out an overflow in y (sum k + sg sum|k| or t + |t|
            // can exceed the f32 range): y * 0 + g1 is NaN exactly when y is inf or NaN, which the
            // bracket below cannot see (a NaN y rounds both ends to the same word)
            g1 = __ffma2_rn(y2, make_float2(0.f, 0.f), g1);
          } else {
            y2 = b2;
#pragma unroll
            for (int i = 0; i < N; ++i) y2 = __ffma2_rn(make_float2(w32[i], w32[i]), k2[i], y2);
            // no vote margin: y * 0 is NaN exactly when y overflowed (inf or NaN), which the bracket
            // below cannot see (a NaN y rounds both bracket ends to the same word)
            g1 = __fmul2_rn(y2, make_float2(0.f, 0.f));
          }
          // bf16 rounding must be certain.  The f32 evaluation error is <= (N + 5) * 2^-24 * S with
          // S = |b| + max w * sum|k|: 3 roundings in k, 1 in w, 1 in y, and N more -- the weighted sum
          // (N roundings, general weights), or for uniform weights (N - 1)/2 each from sum|k| and sum k
          // (weighted by w/2) plus 1 for sg sum|k| + sum k.  So the reference's value lies in
          // [y - c S, y + c S] with c = (N + 7) 2^-24: one 2^-24 S for the rounding of each bracket end
          // (|end| <= (1 + c) S) and one spare (S2 itself is computed short by <= N 2^-24 relative).  RN to
          // bf16 is monotone, so if both ends round to the same bf16 word, so does the reference's value
          // -- the bracket covers the rounding boundaries on both sides of y, including the closer one
          // below a power of two.  The output IS the lower end's word.
          const float2 ylo = __ffma2_rn(make_float2(-kBr, -kBr), S2, y2);
          const float2 yhi = __ffma2_rn(make_float2(kBr, kBr), S2, y2);
          const uint32_t wlo = pack_bf16x2(ylo);
          mx[p] = wlo ^ pack_bf16x2(yhi);
          if constexpr (ERASE == 2) {
            // unscaled squared vote: k^2 must stay normal (|k| >= 2^-63), which S >= 2^-38 guarantees
            // with sr >= 2^-16; g3 = max(S * 2^38 - 1, -S) < 0 exactly for 0 < S < 2^-38 (-0 for S == 0,
            // an all-zero column), and overflow to inf makes a margin NaN
            const float2 g3a = __ffma2_rn(S2, make_float2(0x1p38f, 0x1p38f), make_float2(-1.f, -1.f));
            gm[p] = make_float2(fmin_nan(g1.x, fmaxf(g3a.x, -S2.x)), fmin_nan(g1.y, fmaxf(g3a.y, -S2.y)));
          } else {
            gm[p] = g1;
          }
          outw[p] = wlo;
        }
        float gmin = fmin_nan(gm[0].x, gm[0].y);
#pragma unroll
        for (int q = 1; q < kFastPairs; ++q) gmin = fmin3_nan(gmin, gm[q].x, gm[q].y);
        uint32_t anym = mx[0];
#pragma unroll
        for (int q = 1; q < kFastPairs; ++q) anym |= mx[q];
        if (!(gmin >= 0.f) || anym != 0u) {  // a margin negative or NaN, or a bracket straddling a boundary
          uint32_t slowm = 0;
#pragma unroll
          for (int q = 0; q < kFastPairs; ++q) {
            // per element: a failed vote margin flags only its own element (its pair partner's
            // margin and bracket are independent)
            const uint32_t bad_x = !(gm[q].x >= 0.f), bad_y = !(gm[q].y >= 0.f);
#ifdef RLK_DEBUG_FLAGS
            dbg_vote += bad_x + bad_y;
            dbg_brk += ((mx[q] & 0xffffu) != 0u) + ((mx[q] >> 16) != 0u);
#endif
            slowm |= ((bad_x | ((mx[q] & 0xffffu) != 0u)) << (2 * q)) | ((bad_y | ((mx[q] >> 16) != 0u)) << (2 * q + 1));
          }
          slowbits |= slowm << jit;
        }
        FastVec::store(outp + out_base + le, outw);
      };
      constexpr uint32_t kIters = ELEMS / (kFastElems * kFastCThreads);
      static_assert(kIters * kFastElems * kFastCThreads == ELEMS, "a full stage is a whole number of iterations");
      if (fast_ok && n == ELEMS) {
        // full stage: compile-time trip count, constant smem / global offsets
#pragma unroll
        for (uint32_t it = 0; it < kIters; ++it) vec(tid + it * kFastCThreads, it * kFastElems);
      } else if (fast_ok) {
        uint32_t jit = 0;
        for (uint32_t v = tid; v < nvec; v += kFastCThreads, jit += kFastElems) vec(v, jit);
      }
#ifdef RLK_TIMING_SKIP_PHASE2  // diagnostic builds only (tools/build_variant.py): phase 2 not run
      slowbits = 0;
#endif
      // phase 2a: the flagged elements go to the fix-up queue -- one shared-memory atomic per warp
      // (warp prefix sum of the lanes' counts), then each lane writes its entries
      if (a.fix_q && __any_sync(0xffffffffu, slowbits != 0u)) {
        const uint32_t c = __popc(slowbits);
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        uint32_t base = 0;
        if (lane == 31) base = atomicAdd(&fix_n, tot);
        base = __shfl_sync(0xffffffffu, base, 31);
        if (base + tot <= a.fix_cap) {
          uint32_t slot = base + incl - c;
          while (slowbits) {
            const uint32_t bpos = __ffs(slowbits) - 1;
            slowbits &= slowbits - 1;
            const uint32_t le = (tid + (bpos / kFastElems) * kFastCThreads) * kFastElems + (bpos % kFastElems);
            uint32_t h[2 + N], keep = 0;
            h[0] = reinterpret_cast<const uint16_t*>(sb)[le];
#pragma unroll
            for (int i = 0; i < N; ++i) {
              h[1 + i] = reinterpret_cast<const uint16_t*>(sb + (i + 1) * SB)[le];
              keep |= DROP ? (((uint32_t)bm[i * BMB + (le >> 3)] >> (le & 7)) & 1u) << i : (1u << i);
            }
            h[1 + N] = 0;
            uint4* qe = a.fix_q + ((uint64_t)blockIdx.x * a.fix_cap + slot++) * kFixWords<N>;
            qe[0] = make_uint4(cur.lo | (keep << 24), (uint32_t)(out_base + le), h[0] | (h[1] << 16),
                               N >= 2 ? (h[2] | (h[3] << 16)) : 0u);
            if constexpr (kFixWords<N> > 1) {
              uint32_t r[4] = {0u, 0u, 0u, 0u};
#pragma unroll
              for (int k = 4; k < 2 + N; k += 2) r[(k - 4) / 2] = h[k] | ((k + 1 < 2 + N ? h[k + 1] : 0u) << 16);
              qe[1] = make_uint4(r[0], r[1], r[2], r[3]);
            }
          }
        } else if (lane == 31) {
          atomicSub(&fix_n, tot);  // the queue is full: this warp finishes its elements below
        }
      }
      // phase 2b (queue full, or no queue): exact reference-order evaluation of the recorded elements,
      // read back from the stage; the 2-byte store follows this thread's own vector store of the word
      while (slowbits) {
        const uint32_t bpos = __ffs(slowbits) - 1;
        slowbits &= slowbits - 1;
        const uint32_t le = (tid + (bpos / kFastElems) * kFastCThreads) * kFastElems + (bpos % kFastElems);
        RLK_DCHECK(le < main_elems && off + le < g.len);
        const float be = __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(sb)[le] << 16);
        FArr<N> xe;
        uint32_t keep = 0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          xe.v[i] = __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(sb + (i + 1) * SB)[le] << 16);
          keep |= DROP ? (((uint32_t)bm[i * BMB + (le >> 3)] >> (le & 7)) & 1u) << i : (1u << i);
        }
        if constexpr (ERASE == 1) {
          if (tie_ok) {  // exact sum-vote ties certified in scalar f32
            uint32_t xb[N], fo = 0;
            uint16_t wout;
#pragma unroll
            for (int i = 0; i < N; ++i) xb[i] = reinterpret_cast<const uint16_t*>(sb + (i + 1) * SB)[le];
            const int kind = scalar_resolve<N, ERASE, UNI>(reinterpret_cast<const uint16_t*>(sb)[le], xb, keep,
                                                           sr32, w32, wh32, wmax, tie_ok, &wout, &fo);
            if (kind) {
              if (kind == 2) {
#pragma unroll
                for (int i = 0; i < N; ++i) cnt_er[i] -= (fo >> i) & 1u;
              }
              outp[out_base + le] = wout;
              continue;
            }
          }
        }
        uint32_t nzm, erm;
        const double Y = merge_elem_slow<N>(be, xe, keep, &a, scale, &nzm, &erm);
        if constexpr (kErase) {
          const uint32_t fo = fast_opp_bits<N>(be, xe.v, keep, sr32, ERASE, false);
#pragma unroll
          for (int i = 0; i < N; ++i) cnt_er[i] += ((erm >> i) & 1u) - ((fo >> i) & 1u);
        }
        outp[out_base + le] = (uint16_t)f64_to_bf16_rne(Y);
      }
      // items the fast path cannot certify, and the < 16-byte tail: exact f64 path
      const uint32_t e0 = fast_ok ? main_elems : 0;
      for (uint32_t e = e0 + tid; e < n; e += kFastCThreads) {
        const uint64_t idx = g.start + off + e;
        const double B = load_f64<RLK_BF16>(g.seg->base, idx);
        double X[N];
#pragma unroll
        for (int i = 0; i < N; ++i) X[i] = load_f64<RLK_BF16>(g.seg->expert[i], idx);
        uint32_t keep = (1u << N) - 1u;
        if (DROP) {
          keep = 0;
#pragma unroll
          for (int i = 0; i < N; ++i) keep |= (uint32_t)keep_draw(a.seed[i], jtensor0 + off + e, a.thresh) << i;
        }
        uint32_t nzm, erm;
        const double Y = merge_elem_f64<N>(B, X, keep, a, c, nzm, erm);
#pragma unroll
        for (int i = 0; i < N; ++i) cnt_er[i] += (erm >> i) & 1u;
        (void)nzm;
        store_from_f64<RLK_BF16>(g.out, idx, Y);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&r.empty[s]);
      q.next(r.nstages);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const uint32_t er = __reduce_add_sync(0xffffffffu, cnt_er[i]);
      if (lane == 0 && er) atomicAdd(a.counters + (uint64_t)g.tensor * 2 * N + N + i, (unsigned long long)er);
    }
  }
#ifdef RLK_DEBUG_FLAGS
  {
    const uint32_t v = __reduce_add_sync(0xffffffffu, dbg_vote), b = __reduce_add_sync(0xffffffffu, dbg_brk);
    if (lane == 0 && blockIdx.x < 4) printf("DBG blk %d warp %d vote %u bracket %u\n", (int)blockIdx.x, warp, v, b);
  }
#endif
  if (a.fix_q) {
    asm volatile("bar.sync 2, %0;" ::"n"(kFastCThreads) : "memory");  // every consumer warp has queued
    if (tid == 0) a.fix_count[blockIdx.x] = min(fix_n, a.fix_cap);
  }
}

// Deferred exact path of k_merge_fast: block b finishes the elements merge CTA b queued, one per thread,
// from global memory in the reference's operation order (merge_elem_f64), and replaces the fast loop's
// erased counts for them (fast_opp_bits -> exact).  Same stream, right after the merge.
template <int N, int DROP, int ERASE>
__global__ void __launch_bounds__(256) k_merge_fixup(const __grid_constant__ MergeArgs a) {
  constexpr bool kErase = (ERASE != 0) && (N >= 2);
  constexpr float kKS = ERASE == 2 ? 1.f : 0x1p24f;  // the fast kernel's scaled domain (sr32 for fast_opp_bits)
  // blockIdx.y splits one CTA's queue over several blocks: every element is a chain of dependent
  // global loads (segment -> pointers -> data), so the kernel needs many threads in flight
  const uint32_t n = a.fix_count[blockIdx.x];
  uint32_t c_seg = 0xffffffffu;  // per-segment constants, reloaded only when the segment changes
  const rlk_fusion_segment* seg = nullptr;
  uint32_t t = 0;
  ElemConsts c;
  float sr32[N];
  for (uint32_t k = blockIdx.y * blockDim.x + threadIdx.x; k < n; k += blockDim.x * gridDim.y) {
    const uint4* q = a.fix_q + ((uint64_t)blockIdx.x * a.fix_cap + k) * kFixWords<N>;
    uint32_t h[2 * 4 * kFixWords<N>];  // the entry as u32 words
    {
      const uint4 q0 = q[0];
      h[0] = q0.x; h[1] = q0.y; h[2] = q0.z; h[3] = q0.w;
      if constexpr (kFixWords<N> > 1) {
        const uint4 q1 = q[1];
        h[4] = q1.x; h[5] = q1.y; h[6] = q1.z; h[7] = q1.w;
      }
    }
    auto half = [&](int m) { return (h[2 + m / 2] >> (16 * (m & 1))) & 0xffffu; };  // bf16 input m (0 = base)
    const uint32_t keep = h[0] >> 24;
    const uint64_t idx = h[1];
    if ((h[0] & 0xffffffu) != c_seg) {
      c_seg = h[0] & 0xffffffu;
      seg = a.plan.segs + c_seg;
      t = seg->tensor;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        c.scale[i] = a.scale[(uint64_t)t * N + i];
        sr32[i] = (float)(DROP ? c.scale[i] / a.keep_prob : c.scale[i]) * kKS;
      }
    }
    float xf[N];
    double X[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      xf[i] = __uint_as_float(half(1 + i) << 16);
      X[i] = (double)xf[i];
    }
    const float bf = __uint_as_float(half(0) << 16);
    uint32_t nzm, erm;
    const double Y = merge_elem_f64<N>((double)bf, X, keep, a, c, nzm, erm);
    reinterpret_cast<uint16_t*>(seg->out)[idx] = f64_to_bf16_rne(Y);
    if constexpr (kErase) {
      const uint32_t fo = fast_opp_bits<N>(bf, xf, keep, sr32, ERASE, false);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int corr = (int)((erm >> i) & 1u) - (int)((fo >> i) & 1u);
        if (corr) atomicAdd(a.counters + (uint64_t)t * 2 * N + N + i, (unsigned long long)(long long)corr);
      }
    }
  }
}

// ------------------------------------------------------------------ host-side launch helpers
// K3 work-unit split for layouts with fewer items than ~2 waves of CTAs (config 1: 154 items on 296
// CTA slots): 2^s units per item, at most one ring stage per unit apart (`stages_per_item`), so every
// CTA slot gets work.  Large layouts keep whole items (s = 0).
// Work units of 65536 >> s elements for layouts with few items: split until there are >= 8 units per
// CTA (the CTAs stride over units, so the last round is at most 1/8 of the work: config 1's 153 items
// over 296 CTAs were 2 or 3 whole-item halves per CTA, 27% idle), keeping >= 2 ring stages per unit.
static uint32_t sub_shift_for(uint32_t n_items, uint32_t cap, uint32_t stages_per_item) {
  uint32_t s = 0;
  while (s < 5 && (uint64_t(n_items) << s) < 8ull * cap && (1u << (s + 1)) <= stages_per_item) ++s;
  return s;
}

template <int N>
static void stage_geometry(int esz, bool bitmap, uint32_t& stage_bytes, uint32_t& nstages) {
  const uint32_t sb = StreamBytes<N>::v;
  const uint32_t elems = sb / esz;
  stage_bytes = (N + 1) * sb + (bitmap ? N * (elems / 8) : 0);
  stage_bytes = (stage_bytes + 127) & ~127u;
  nstages = (kSmemBudget - 1024) / stage_bytes;
  if (nstages > 8) nstages = 8;
}

template <typename K>
static int ensure_smem(K kernel, uint32_t bytes) {
  return cuda_status(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
                     "cudaFuncSetAttribute");
}

template <int DT, int N>
static int launch_sumsq(SumsqArgs& a, cudaStream_t s) {
  uint32_t sb, ns;
  stage_geometry<N>(Elem<DT>::size, a.counters && a.dropout_mode == 2, sb, ns);
  ns = std::max<uint32_t>(2u, std::min<uint32_t>(ns / 2, 4u));  // two CTAs per SM
  a.stage_bytes = sb;
  a.nstages = ns;
  const uint32_t smem = 1024 + sb * ns;
  auto kern = k_sumsq<DT, N>;
  if constexpr (DT == RLK_F32) {
    if (!a.delta_mode && !(a.counters && a.dropout_mode == 1))
      kern = !a.counters ? k_sumsq<DT, N, 0> : (a.dropout_mode == 2 ? k_sumsq<DT, N, 2> : k_sumsq<DT, N, 1>);
  }
  if constexpr (DT == RLK_BF16 && N <= 4) {
    // pair mode with no inline dropout draws: the bf16 fast kernel
    if (!a.delta_mode && !(a.counters && a.dropout_mode == 1)) {
      kern = !a.counters ? k_sumsq_bf16<N, 0> : (a.dropout_mode == 2 ? k_sumsq_bf16<N, 2> : k_sumsq_bf16<N, 1>);
    }
  }
  int st = ensure_smem(kern, smem);
  if (st) return st;
  uint32_t grid = std::min<uint32_t>(a.plan.n_items, 2u * (uint32_t)sm_count());
  kern<<<grid, kThreads, smem, s>>>(a);
  return launch_status("rlk_fusion_sumsq");
}

template <int N, int DROP, int ERASE, bool UNI = false>
static int launch_merge_fast(MergeArgs& a, cudaStream_t s) {
  uint32_t sb = (N + 1) * kFastSB + (DROP ? N * (kFastSB / 2 / 8) : 0);
  sb = (sb + 127) & ~127u;
  a.stage_bytes = sb;
  a.nstages = std::min<uint32_t>(8, (kSmemBudget / kFastCtas - 1024) / sb);
  const uint32_t smem = 1024 + a.stage_bytes * a.nstages;
  auto kern = k_merge_fast<N, DROP, ERASE, UNI>;
  int st = ensure_smem(kern, smem);
  if (st) return st;
  const uint32_t cap = kFastCtas * (uint32_t)sm_count();
  a.sub_shift = sub_shift_for(a.plan.n_items, cap, kItem / kFastSB * 2);
  uint32_t grid = std::min<uint32_t>(a.plan.n_items << a.sub_shift, cap);
  if (a.fix_q) {
    a.fix_cap = (uint32_t)std::min<uint64_t>(a.fix_cap_total / kFixWords<N> / grid, 0xffffffffu);
    if (a.fix_cap == 0 || a.plan.n_segs >= (1u << 24)) a.fix_q = nullptr;
  }
  kern<<<grid, kFastThreads, smem, s>>>(a);
  if (int st = launch_status("rlk_fusion_merge")) return st;
  if (a.fix_q) {
    k_merge_fixup<N, DROP, ERASE><<<dim3(grid, 8), 256, 0, s>>>(a);
    return launch_status("rlk_fusion_merge (fix-up)");
  }
  return RLK_OK;
}

template <int N>
static int dispatch_fast(MergeArgs& a, cudaStream_t s) {
  const int ec = N >= 2 ? a.erase_mode : 0;
  bool uni = true;
  for (int i = 1; i < N; ++i) uni = uni && a.w[i] == a.w[0];
  if (a.dropout_mode == 2) {
    if (ec == 1) return uni ? launch_merge_fast<N, 2, 1, true>(a, s) : launch_merge_fast<N, 2, 1>(a, s);
    if (ec == 2) return uni ? launch_merge_fast<N, 2, 2, true>(a, s) : launch_merge_fast<N, 2, 2>(a, s);
    return launch_merge_fast<N, 2, 0>(a, s);
  }
  if (ec == 1) return uni ? launch_merge_fast<N, 0, 1, true>(a, s) : launch_merge_fast<N, 0, 1>(a, s);
  if (ec == 2) return uni ? launch_merge_fast<N, 0, 2, true>(a, s) : launch_merge_fast<N, 0, 2>(a, s);
  return launch_merge_fast<N, 0, 0>(a, s);
}

template <int DTI, int DTO, int N>
static int launch_merge(MergeArgs& a, cudaStream_t s) {
  uint32_t sb, ns;
  stage_geometry<N>(Elem<DTI>::size, a.dropout_mode == 2, sb, ns);
  a.stage_bytes = sb;
  a.nstages = ns;
  if constexpr (DTI == RLK_BF16 && DTO == RLK_BF16 && N <= 4) {
    if (a.fast && !a.delta_mode && a.with_base && a.dropout_mode != 1) return dispatch_fast<N>(a, s);
  }
  // two CTAs per SM (N <= 5; more experts would spill): the reference-order f64 arithmetic is
  // latency-bound, so it needs the warps
  constexpr uint32_t ctas = N <= 5 ? 2u : 1u;
  if (ctas == 2) a.nstages = ns = std::max<uint32_t>(2u, std::min<uint32_t>(ns / 2, 4u));
  const uint32_t smem = 1024 + sb * ns;
  auto kern = k_merge<DTI, DTO, N>;
  if constexpr (DTI == RLK_F32 && DTO == RLK_F32 && N >= 2 && N <= 4) {
    // f32 checkpoints: the compile-time-mode kernel (same arithmetic; exact_path keeps the generic one)
    if (a.fast && !a.delta_mode && a.with_base && a.dropout_mode != 1 && a.erase_mode >= 0 && a.erase_mode <= 2) {
      const int d = a.dropout_mode == 2 ? 1 : 0, e = a.erase_mode;
      kern = d ? (e == 0 ? k_merge<DTI, DTO, N, 4> : e == 1 ? k_merge<DTI, DTO, N, 5> : k_merge<DTI, DTO, N, 6>)
               : (e == 0 ? k_merge<DTI, DTO, N, 1> : e == 1 ? k_merge<DTI, DTO, N, 2> : k_merge<DTI, DTO, N, 3>);
    }
  }
  int st = ensure_smem(kern, smem);
  if (st) return st;
  const uint32_t cap = ctas * (uint32_t)sm_count();
  a.sub_shift = sub_shift_for(a.plan.n_items, cap, kItem / StreamBytes<N>::v * Elem<DTI>::size);
  uint32_t grid = std::min<uint32_t>(a.plan.n_items << a.sub_shift, cap);
  kern<<<grid, kThreads, smem, s>>>(a);
  return launch_status("rlk_fusion_merge");
}

template <int DT>
static int dispatch_sumsq_n(int n, SumsqArgs& a, cudaStream_t s) {
  switch (n) {
    case 1: return launch_sumsq<DT, 1>(a, s);
    case 2: return launch_sumsq<DT, 2>(a, s);
    case 3: return launch_sumsq<DT, 3>(a, s);
    case 4: return launch_sumsq<DT, 4>(a, s);
    case 5: return launch_sumsq<DT, 5>(a, s);
    case 6: return launch_sumsq<DT, 6>(a, s);
    case 7: return launch_sumsq<DT, 7>(a, s);
    case 8: return launch_sumsq<DT, 8>(a, s);
  }
  set_error("expert count %d not supported (1..%d)", n, RLK_MAX_EXPERTS);
  return RLK_ERR_UNSUPPORTED;
}

template <int DTI, int DTO>
static int dispatch_merge_n(int n, MergeArgs& a, cudaStream_t s) {
  switch (n) {
    case 1: return launch_merge<DTI, DTO, 1>(a, s);
    case 2: return launch_merge<DTI, DTO, 2>(a, s);
    case 3: return launch_merge<DTI, DTO, 3>(a, s);
    case 4: return launch_merge<DTI, DTO, 4>(a, s);
    case 5: return launch_merge<DTI, DTO, 5>(a, s);
    case 6: return launch_merge<DTI, DTO, 6>(a, s);
    case 7: return launch_merge<DTI, DTO, 7>(a, s);
    case 8: return launch_merge<DTI, DTO, 8>(a, s);
  }
  set_error("expert count %d not supported (1..%d)", n, RLK_MAX_EXPERTS);
  return RLK_ERR_UNSUPPORTED;
}

template <int DTI>
static int dispatch_merge_out(int dto, int n, MergeArgs& a, cudaStream_t s) {
  switch (dto) {
    case RLK_BF16: return dispatch_merge_n<DTI, RLK_BF16>(n, a, s);
    case RLK_F32: return dispatch_merge_n<DTI, RLK_F32>(n, a, s);
    case RLK_F64: return dispatch_merge_n<DTI, RLK_F64>(n, a, s);
  }
  set_error("bad output dtype %d", dto);
  return RLK_ERR_INVALID;
}

}  // namespace rlk

using namespace rlk;

extern "C" {

int rlk_fusion_sumsq(const rlk_fusion_plan* plan, int n_experts, int dtype, int delta_mode, double* partials,
                     unsigned long long* nz_counters, int dropout_mode, const uint64_t* child_seeds, uint64_t thresh,
                     const uint32_t* bitmap, uint64_t words_per_row, void* stream) {
  RLK_REQUIRE(plan != nullptr && partials != nullptr, "rlk_fusion_sumsq: NULL argument");
  RLK_REQUIRE(n_experts >= 1 && n_experts <= RLK_MAX_EXPERTS, "rlk_fusion_sumsq: bad expert count %d", n_experts);
  RLK_REQUIRE(dropout_mode >= 0 && dropout_mode <= 2, "rlk_fusion_sumsq: bad dropout mode %d", dropout_mode);
  RLK_REQUIRE(!nz_counters || dropout_mode == 0 || child_seeds, "rlk_fusion_sumsq: dropout needs child seeds");
  RLK_REQUIRE(!nz_counters || dropout_mode != 2 || (bitmap && words_per_row % 4 == 0),
              "rlk_fusion_sumsq: bitmap mode needs a bitmap with 16-byte rows");
  if (plan->n_items == 0) return RLK_OK;
  RLK_REQUIRE(plan->segs && plan->seg_item_prefix && plan->n_segs > 0, "rlk_fusion_sumsq: empty plan");
  SumsqArgs a;
  memset(&a, 0, sizeof(a));
  a.plan = *plan;
  a.partials = partials;
  a.counters = nz_counters;
  a.bitmap = bitmap;
  a.words_per_row = words_per_row;
  for (int i = 0; i < n_experts; ++i) a.seed[i] = child_seeds ? child_seeds[i] : 0;
  a.thresh = thresh;
  a.delta_mode = delta_mode;
  a.dropout_mode = nz_counters ? dropout_mode : 0;
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case RLK_BF16: return dispatch_sumsq_n<RLK_BF16>(n_experts, a, s);
    case RLK_F32: return dispatch_sumsq_n<RLK_F32>(n_experts, a, s);
    case RLK_F64: return dispatch_sumsq_n<RLK_F64>(n_experts, a, s);
  }
  set_error("rlk_fusion_sumsq: bad dtype %d", dtype);
  return RLK_ERR_INVALID;
}

int rlk_fusion_finalize(const double* partials, const uint32_t* tensor_items, uint32_t n_tensors, int n_experts,
                        int target_mode, double target_value, double* sumsq, double* scale, int32_t* status,
                        void* stream) {
  RLK_REQUIRE(n_experts >= 1 && n_experts <= RLK_MAX_EXPERTS, "rlk_fusion_finalize: bad expert count %d", n_experts);
  RLK_REQUIRE(target_mode >= 0 && target_mode <= 2, "rlk_fusion_finalize: bad target mode %d", target_mode);
  if (n_tensors == 0) return RLK_OK;
  RLK_REQUIRE(partials && tensor_items && sumsq && scale && status, "rlk_fusion_finalize: NULL argument");
  const int warps = 8;
  const uint32_t grid = (n_tensors + warps - 1) / warps;
  k_finalize<<<grid, warps * 32, 0, (cudaStream_t)stream>>>(partials, tensor_items, n_tensors, n_experts,
                                                            target_mode, target_value, sumsq, scale, status);
  return launch_status("rlk_fusion_finalize");
}

int rlk_fusion_mask_bitmap_range(const uint64_t* child_seeds, int n_experts, uint64_t thresh, uint64_t bit_lo,
                                 uint64_t bit_hi, uint32_t* bitmap, uint64_t words_per_row, void* stream) {
  RLK_REQUIRE(n_experts >= 1 && n_experts <= RLK_MAX_EXPERTS, "rlk_fusion_mask_bitmap: bad expert count %d",
              n_experts);
  RLK_REQUIRE(child_seeds && bitmap, "rlk_fusion_mask_bitmap: NULL argument");
  RLK_REQUIRE(bit_lo % 32 == 0 && bit_lo <= bit_hi, "rlk_fusion_mask_bitmap: bad bit range");
  RLK_REQUIRE(words_per_row * 32 >= bit_hi, "rlk_fusion_mask_bitmap: row too short");
  if (bit_hi == bit_lo) return RLK_OK;
  ulonglong4 lo = make_ulonglong4(0, 0, 0, 0), hi = make_ulonglong4(0, 0, 0, 0);
  for (int i = 0; i < n_experts; ++i) (i < 4 ? (&lo.x)[i] : (&hi.x)[i - 4]) = child_seeds[i];
  const uint64_t words = (bit_hi - bit_lo + 31) / 32;
  const uint64_t blocks = (words + 255) / 256;
  const uint32_t gx = (uint32_t)std::min<uint64_t>(blocks, (uint64_t)sm_count() * 16 / n_experts + 1);
  const uint64_t t64 = thresh << 11;  // thresh == 0 (p = 0): t64 == 0 keeps every draw in any mode
  auto kern = (t64 & 0xffffffffull) != 0 ? k_mask_bitmap<0>
              : ((t64 >> 32) & 1u) ? k_mask_bitmap<1> : k_mask_bitmap<2>;
  kern<<<dim3(gx, n_experts), 256, 0, (cudaStream_t)stream>>>(lo, hi, n_experts, thresh, bit_lo / 32, bit_hi, bitmap,
                                                              words_per_row);
  return launch_status("rlk_fusion_mask_bitmap");
}

int rlk_fusion_mask_bitmap(const uint64_t* child_seeds, int n_experts, uint64_t thresh, uint64_t n_bits,
                           uint32_t* bitmap, uint64_t words_per_row, void* stream) {
  return rlk_fusion_mask_bitmap_range(child_seeds, n_experts, thresh, 0, n_bits, bitmap, words_per_row, stream);
}

int rlk_fusion_merge(const rlk_fusion_plan* plan, int n_experts, int dtype_in, int dtype_out, int delta_mode,
                     const double* scale, const double* weights, int dropout_mode, const uint64_t* child_seeds,
                     uint64_t thresh, double keep_prob, const uint32_t* bitmap, uint64_t words_per_row,
                     int erase_mode, unsigned long long* counters, int exact_path, void* stream) {
  return rlk_fusion_merge_ws(plan, n_experts, dtype_in, dtype_out, delta_mode, scale, weights, dropout_mode,
                             child_seeds, thresh, keep_prob, bitmap, words_per_row, erase_mode, counters, exact_path,
                             nullptr, 0, stream);
}

int rlk_fusion_merge_ws(const rlk_fusion_plan* plan, int n_experts, int dtype_in, int dtype_out, int delta_mode,
                        const double* scale, const double* weights, int dropout_mode, const uint64_t* child_seeds,
                        uint64_t thresh, double keep_prob, const uint32_t* bitmap, uint64_t words_per_row,
                        int erase_mode, unsigned long long* counters, int exact_path, void* workspace,
                        uint64_t workspace_bytes, void* stream) {
  RLK_REQUIRE(plan && scale && weights && counters, "rlk_fusion_merge: NULL argument");
  RLK_REQUIRE(n_experts >= 1 && n_experts <= RLK_MAX_EXPERTS, "rlk_fusion_merge: bad expert count %d", n_experts);
  RLK_REQUIRE(dropout_mode >= 0 && dropout_mode <= 2, "rlk_fusion_merge: bad dropout mode %d", dropout_mode);
  RLK_REQUIRE(erase_mode >= 0 && erase_mode <= 2, "rlk_fusion_merge: bad erase mode %d", erase_mode);
  RLK_REQUIRE(dropout_mode == 0 || child_seeds, "rlk_fusion_merge: dropout needs child seeds");
  RLK_REQUIRE(dropout_mode != 2 || (bitmap && words_per_row % 4 == 0),
              "rlk_fusion_merge: bitmap mode needs a bitmap with 16-byte rows");
  RLK_REQUIRE(dropout_mode == 0 || (keep_prob > 0.0 && keep_prob <= 1.0), "rlk_fusion_merge: bad keep_prob");
  if (plan->n_items == 0) return RLK_OK;
  MergeArgs a{};
  memset(&a, 0, sizeof(a));
  a.plan = *plan;
  a.scale = scale;
  for (int i = 0; i < n_experts; ++i) {
    a.w[i] = weights[i];
    a.seed[i] = child_seeds ? child_seeds[i] : 0;
  }
  a.thresh = thresh;
  a.keep_prob = keep_prob;
  a.inv_keep = 1.0 / keep_prob;
  a.bitmap = bitmap;
  a.words_per_row = words_per_row;
  a.counters = counters;
  a.dropout_mode = dropout_mode;
  a.erase_mode = erase_mode;
  a.delta_mode = delta_mode & 1;
  a.with_base = (delta_mode & 1) ? ((delta_mode >> 1) & 1) : 1;
  a.fast = exact_path ? 0 : 1;
  // workspace: [per-CTA queue lengths: 4 KiB | queue entries (8 B each)]
  if (workspace && workspace_bytes > RLK_MERGE_WS_HEADER && ((uintptr_t)workspace & 15u) == 0) {
    a.fix_count = (uint32_t*)workspace;
    a.fix_q = (uint4*)((char*)workspace + RLK_MERGE_WS_HEADER);
    a.fix_cap_total = (workspace_bytes - RLK_MERGE_WS_HEADER) / sizeof(uint4);  // in uint4 words
  }
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype_in) {
    case RLK_BF16: return dispatch_merge_out<RLK_BF16>(dtype_out, n_experts, a, s);
    case RLK_F32: return dispatch_merge_out<RLK_F32>(dtype_out, n_experts, a, s);
    case RLK_F64: return dispatch_merge_out<RLK_F64>(dtype_out, n_experts, a, s);
  }
  set_error("rlk_fusion_merge: bad input dtype %d", dtype_in);
  return RLK_ERR_INVALID;
}

}  // extern "C"
