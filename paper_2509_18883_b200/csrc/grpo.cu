// GRPO token objective kernels for sm_100a: K4 forward (online log-sum-exp over the vocab row + token
// gather + TIS + triplet clip epilogue) and K5 backward (coef * (onehot - softmax)).
//
// Reference (pkg/src/rolloutlab/):
//   log_token_dist        toy_env.py:157-175   z / T; lse = max + log(sum(exp(z - max))); z - lse
//   _triplet_value_slope  objective.py:133-150
//   tis_weight            objective.py:161-165 min(exp(logp_train - logp_infer), cap)
//   objective_value       objective.py:230-250 r = exp(logp - logp_train); g_sum += w * value
//   objective_gradient    objective.py:253-283 coef = norm * w * slope * r / T; row -= coef * p; row[tok] += coef
//
// A logits row (V = 131072 bf16 = 256 KiB) is streamed through a TMA bulk-copy ring by one producer
// lane; eight consumer warps keep a per-thread (max, sum 2^(z*c - max*c)) pair in f32 (c = log2(e) / T,
// MUFU.EX2 per logit), combined with shuffles at the end of the row.  The epilogue runs in f64.
#include <type_traits>

#include "common.cuh"
#include "capi_internal.h"
#include "pipeline.cuh"

namespace rlk {

constexpr uint32_t kRowStageBytes = 32768;
constexpr uint32_t kRowStages = 6;
// 16 consumer warps + 1 producer warp: the per-logit chain (max, FFMA, MUFU.EX2, FADD) is short, so
// latency hiding needs warps (profiles/r01: 8 warps gave IPC 1.6 and 52% of HBM peak)
constexpr int kGW = 16;
constexpr int kGT = kGW * 32;
constexpr int kGThreads = kGT + 32;
__device__ __forceinline__ void gbar_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kGT) : "memory"); }
constexpr double kLog2e = 1.4426950408889634074;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int DT> struct RowVec;
template <> struct RowVec<RLK_BF16> {
  static constexpr int n = 8;
  __device__ static void f32(const uint4& w, float* o) {
    o[0] = bf16_lo(w.x); o[1] = bf16_hi(w.x); o[2] = bf16_lo(w.y); o[3] = bf16_hi(w.y);
    o[4] = bf16_lo(w.z); o[5] = bf16_hi(w.z); o[6] = bf16_lo(w.w); o[7] = bf16_hi(w.w);
  }
};
template <> struct RowVec<RLK_F32> {
  static constexpr int n = 4;
  __device__ static void f32(const uint4& w, float* o) {
    o[0] = __uint_as_float(w.x); o[1] = __uint_as_float(w.y); o[2] = __uint_as_float(w.z); o[3] = __uint_as_float(w.w);
  }
};
template <> struct RowVec<RLK_F64> {
  static constexpr int n = 2;
  __device__ static void f64(const uint4& w, double* o) {
    o[0] = __hiloint2double((int)w.y, (int)w.x);
    o[1] = __hiloint2double((int)w.w, (int)w.z);
  }
};

// Producer lane: stream the rows this CTA owns (row = blockIdx.x + k * gridDim.x, skipping inactive
// rows) through the ring in kRowStageBytes chunks (16-byte multiples; the <16-byte tail is read by
// consumers from global memory).
template <typename Active, typename Addr>
__device__ void produce_rows(const Ring& r, uint64_t n_rows, uint64_t row_bytes, Active active, Addr addr) {
  const uint64_t pol = policy_evict_first();
  RingPos q;
  for (uint64_t row = blockIdx.x; row < n_rows; row += gridDim.x) {
    if (!active(row)) continue;
    const char* src = addr(row);
    for (uint64_t off = 0; off < row_bytes; off += r.stage_bytes) {
      const uint32_t bytes = (uint32_t)umin64((uint64_t)r.stage_bytes, row_bytes - off);
      const uint32_t main_bytes = bytes & ~15u;
      const uint32_t s = q.s, ph = q.ph;
      mbar_wait(&r.empty[s], ph ^ 1u);
      if (main_bytes) {
        mbar_arrive_expect_tx(&r.full[s], main_bytes);
        bulk_g2s(r.buf + s * r.stage_bytes, src + off, main_bytes, &r.full[s], pol);
      } else {
        mbar_arrive(&r.full[s]);
      }
      q.next(r.nstages);
    }
  }
}

// ------------------------------------------------------------------ triplet clip (objective.py:133-150)
struct TripletOut { double value, slope; };
__device__ __forceinline__ TripletOut triplet(double r, double adv, const rlk_clip& c) {
  const double lo = 1.0 - c.eps_neg_low, hi = 1.0 + c.eps_pos_high;
  const double clipped = fmin(fmax(r, lo), hi);
  const double clip_slope = (lo <= r && r <= hi) ? 1.0 : 0.0;
  const double raw = __dmul_rn(r, adv);
  const double capped = __dmul_rn(clipped, adv);
  double inner, islope;
  if (raw <= capped) { inner = raw; islope = adv; }
  else { inner = capped; islope = __dmul_rn(adv, clip_slope); }
  if (c.guard_positive && adv > 0.0) return {inner, islope};
  const double floor_v = __dmul_rn(c.eps_neg_high, adv);
  if (inner >= floor_v) return {inner, islope};
  return {floor_v, 0.0};
}

// log-sum-exp of z / T for a row read straight from global memory (unaligned rows; f64 math).
template <int DT>
__device__ double row_lse_global(const char* rowp, uint64_t V, double T, double* red_m, double* red_s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double m = -INFINITY, sum = 0.0;
  for (uint64_t v = threadIdx.x; v < V; v += kGT) {
    const double z = load_f64<DT>(rowp, v);
    const double zt = T == 1.0 ? z : __ddiv_rn(z, T);
    if (zt > m) { sum = sum * exp(m - zt); m = zt; }
    sum += exp(zt - m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, sum, o);
    const double M = fmax(m, om);
    sum = (M == -INFINITY) ? 0.0 : sum * exp(m - M) + os * exp(om - M);
    m = M;
  }
  if (lane == 0) { red_m[warp] = m; red_s[warp] = sum; }
  gbar_sync();
  double M = red_m[0];
  for (int w = 1; w < kGW; ++w) M = fmax(M, red_m[w]);
  double S = 0.0;
  for (int w = 0; w < kGW; ++w) S += red_m[w] == -INFINITY ? 0.0 : red_s[w] * exp(red_m[w] - M);
  gbar_sync();
  return M + log(S);
}

struct FwdArgs {
  const char* logits;
  uint64_t n_rows, vocab, row_stride;
  const int64_t* row_index;
  const int32_t* tokens;
  const double* lp_train;
  const double* lp_infer;
  const int32_t* sample;
  const double* adv;
  const uint8_t* use;
  const double* temp;
  const double* norm;
  rlk_clip clip;
  double *logp, *lse, *term, *coef;
  int32_t* flags;
};

// f64 epilogue for one token given its natural-log lse (thread-level).
template <int DT>
__device__ void fwd_epilogue(const FwdArgs& a, uint64_t row, const char* rowp, double lse) {
  const int32_t s = a.sample[row];
  const double T = a.temp[s];
  const int32_t tok = a.tokens[row];
  if (tok < 0 || (uint64_t)tok >= a.vocab) {
    atomicOr(a.flags, 2);
    if (a.logp) a.logp[row] = nan("");
    if (a.lse) a.lse[row] = lse;
    a.term[row] = 0.0;
    a.coef[row] = 0.0;
    return;
  }
  const double z = load_f64<DT>(rowp, (uint64_t)tok);
  const double zt = (T == 1.0) ? z : __ddiv_rn(z, T);  // toy_env.py:168-171
  const double logp = __dsub_rn(zt, lse);
  const double lt = a.lp_train[row], li = a.lp_infer[row];
  const double r = exp(__dsub_rn(logp, lt));                                // objective.py:245
  const double w = fmin(exp(__dsub_rn(lt, li)), a.clip.tis_cap);           // objective.py:161-165
  const TripletOut tv = triplet(r, a.adv[s], a.clip);                       // objective.py:247
  if (!isfinite(logp)) atomicOr(a.flags, 1);
  if (a.logp) a.logp[row] = logp;
  if (a.lse) a.lse[row] = lse;
  a.term[row] = __dmul_rn(w, tv.value);
  // objective.py:279: coef = norm * w * slope * r_theta / tau (left to right)
  a.coef[row] = __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(a.norm[s], w), tv.slope), r), T);
}

template <int DT>
__global__ void __launch_bounds__(kGThreads, 1) k_grpo_fwd(FwdArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int ESZ = Elem<DT>::size;
  constexpr int VEC = 16 / ESZ;
  const Ring r = ring_setup(smem, kRowStageBytes, kRowStages, kGW);
  const uint64_t row_bytes = a.vocab * ESZ;
  auto active = [&](uint64_t row) { return a.use[a.sample[row]] != 0; };
  auto addr = [&](uint64_t row) {
    const uint64_t rr = a.row_index ? (uint64_t)a.row_index[row] : row;
    return a.logits + rr * a.row_stride * ESZ;
  };
  // rows whose start is not 16-byte aligned (tiny toy vocabularies) bypass the TMA ring
  auto streamed = [&](uint64_t row) { return active(row) && ((uintptr_t)addr(row) & 15u) == 0; };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  if (warp == kGW) {
    if (lane == 0) produce_rows(r, a.n_rows, row_bytes, streamed, addr);
    return;
  }
  __shared__ double red_m[kGW], red_s[kGW];
  RingPos q;
  for (uint64_t row = blockIdx.x; row < a.n_rows; row += gridDim.x) {
    if (!active(row)) {
      if (tid == 0) {
        if (a.logp) a.logp[row] = 0.0;
        if (a.lse) a.lse[row] = 0.0;
        a.term[row] = 0.0;
        a.coef[row] = 0.0;
      }
      continue;
    }
    const char* rowp = addr(row);
    const double T = a.temp[a.sample[row]];
    double lse;
    if (((uintptr_t)rowp & 15u) != 0) {
      lse = row_lse_global<DT>(rowp, a.vocab, T, red_m, red_s);
    } else if constexpr (DT == RLK_F64) {
      // f64 path: online max / sum of exp(z/T - m) with exact division (toy_env.py:168-174)
      double m = -INFINITY, sum = 0.0;
      for (uint64_t off = 0; off < row_bytes; off += r.stage_bytes) {
        const uint32_t bytes = (uint32_t)umin64((uint64_t)r.stage_bytes, row_bytes - off);
        const uint32_t main_bytes = bytes & ~15u;
        const uint32_t s = q.s, ph = q.ph;
        mbar_wait(&r.full[s], ph);
        const uint8_t* sb = r.buf + s * r.stage_bytes;
        for (uint32_t v = tid; v < main_bytes / 16; v += kGT) {
          double z[2];
          RowVec<RLK_F64>::f64(lds128(sb + v * 16), z);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double zt = T == 1.0 ? z[e] : __ddiv_rn(z[e], T);
            if (zt > m) { sum = sum * exp(m - zt); m = zt; }
            sum += exp(zt - m);
          }
        }
        for (uint32_t e = main_bytes / 8 + tid; e < bytes / 8; e += kGT) {
          const double z = load_f64<DT>(rowp, off / 8 + e);
          const double zt = T == 1.0 ? z : __ddiv_rn(z, T);
          if (zt > m) { sum = sum * exp(m - zt); m = zt; }
          sum += exp(zt - m);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&r.empty[s]);
        q.next(r.nstages);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, sum, o);
        const double M = fmax(m, om);
        sum = (M == -INFINITY) ? 0.0 : sum * exp(m - M) + os * exp(om - M);
        m = M;
      }
      if (lane == 0) { red_m[warp] = m; red_s[warp] = sum; }
      gbar_sync();
      double M = red_m[0];
      for (int w = 1; w < kGW; ++w) M = fmax(M, red_m[w]);
      double S = 0.0;
      for (int w = 0; w < kGW; ++w) S += red_m[w] == -INFINITY ? 0.0 : red_s[w] * exp(red_m[w] - M);
      lse = M + log(S);
      gbar_sync();
    } else {
      // f32 path in the log2 domain: x = z * c, c = log2(e) / T; one MUFU.EX2 per logit.
      const float c = (float)(kLog2e / T);
      float mz = -INFINITY, sum = 0.f, sum2 = 0.f, nb = INFINITY;
      for (uint64_t off = 0; off < row_bytes; off += r.stage_bytes) {
        const uint32_t bytes = (uint32_t)umin64((uint64_t)r.stage_bytes, row_bytes - off);
        const uint32_t main_bytes = bytes & ~15u;
        const uint32_t s = q.s, ph = q.ph;
        mbar_wait(&r.full[s], ph);
        const uint8_t* sb = r.buf + s * r.stage_bytes;
        const uint32_t nvec = main_bytes / 16;
        for (uint32_t v = tid; v < nvec; v += kGT) {
          float z[VEC];
          RowVec<DT>::f32(lds128(sb + v * 16), z);
          float lm = fmaxf(z[0], z[1]);
#pragma unroll
          for (int e = 2; e < VEC; e += 2) lm = fmaxf(lm, fmaxf(z[e], z[e + 1]));
          if (lm > mz) {  // new running max: rescale (rare after the first vectors of a row)
            const float f = ex2_approx((mz - lm) * c);
            sum *= f;
            sum2 *= f;
            mz = lm;
            nb = -mz * c;
          }
#pragma unroll
          for (int e = 0; e < VEC; e += 2) {
            sum += ex2_approx(fmaf(z[e], c, nb));
            sum2 += ex2_approx(fmaf(z[e + 1], c, nb));
          }
        }
        for (uint32_t e = main_bytes / ESZ + tid; e < bytes / ESZ; e += kGT) {
          const float z = (float)load_f64<DT>(rowp, off / ESZ + e);
          if (z > mz) {
            const float f = ex2_approx((mz - z) * c);
            sum *= f;
            sum2 *= f;
            mz = z;
            nb = -mz * c;
          }
          sum += ex2_approx(fmaf(z, c, nb));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&r.empty[s]);
        q.next(r.nstages);
      }
      sum += sum2;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, mz, o), os = __shfl_xor_sync(0xffffffffu, sum, o);
        const float M = fmaxf(mz, om);
        sum = (M == -INFINITY) ? 0.f : sum * ex2_approx((mz - M) * c) + os * ex2_approx((om - M) * c);
        mz = M;
      }
      if (lane == 0) { red_m[warp] = mz; red_s[warp] = sum; }
      gbar_sync();
      double M = red_m[0];
      for (int w = 1; w < kGW; ++w) M = fmax(M, red_m[w]);
      double S = 0.0;
      for (int w = 0; w < kGW; ++w)
        S += red_m[w] == -INFINITY ? 0.0 : red_s[w] * exp2((red_m[w] - M) * (kLog2e / T));
      // lse of z/T (natural log): max/T + ln(S)
      lse = (T == 1.0 ? M : M / T) + log(S);
      gbar_sync();
    }
    if (tid == 0) fwd_epilogue<DT>(a, row, rowp, lse);
  }
}

// ------------------------------------------------------------------ K4 split form (bf16 / f32)
// K4a streams every row and leaves per-(row, warp) partials (max z, sum 2^((z - max) c)) in a
// workspace -- no block-level synchronisation anywhere in the streaming loop; K4b combines the
// kGW partials of a row in f64 and runs the epilogue, one thread per row.
#ifndef RLK_K4A_CTAS
#define RLK_K4A_CTAS 2
#endif
constexpr int kK4aCtas = RLK_K4A_CTAS;  // CTAs per SM of the streaming forward (ring split between them)
template <int DT>
__global__ void __launch_bounds__(kGThreads, kK4aCtas) k_grpo_fwd_stream(FwdArgs a, float* __restrict__ ws) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int ESZ = Elem<DT>::size;
  constexpr int VEC = 16 / ESZ;
  const Ring r = ring_setup(smem, kRowStageBytes, kRowStages / kK4aCtas, kGW);
  const uint64_t row_bytes = a.vocab * ESZ;
  auto active = [&](uint64_t row) { return a.use[a.sample[row]] != 0; };
  auto addr = [&](uint64_t row) {
    const uint64_t rr = a.row_index ? (uint64_t)a.row_index[row] : row;
    return a.logits + rr * a.row_stride * ESZ;
  };
  auto streamed = [&](uint64_t row) { return active(row) && ((uintptr_t)addr(row) & 15u) == 0; };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  if (warp == kGW) {
    if (lane == 0) produce_rows(r, a.n_rows, row_bytes, streamed, addr);
    return;
  }
  RingPos q;
  for (uint64_t row = blockIdx.x; row < a.n_rows; row += gridDim.x) {
    if (!active(row)) continue;
    const char* rowp = addr(row);
    const float c = (float)(kLog2e / a.temp[a.sample[row]]);
    float mz = -INFINITY, sum = 0.f, sum2 = 0.f, sum3 = 0.f, sum4 = 0.f, nb = INFINITY;
    auto take = [&](float z) {
      if (z > mz) {
        const float f = ex2_approx((mz - z) * c);
        sum *= f;
        sum2 *= f;
        sum3 *= f;
        sum4 *= f;
        mz = z;
        nb = -mz * c;
      }
      sum += ex2_approx(fmaf(z, c, nb));
    };
    if (((uintptr_t)rowp & 15u) != 0) {
      for (uint64_t v = tid; v < a.vocab; v += kGT) take((float)load_f64<DT>(rowp, v));
    } else {
      for (uint64_t off = 0; off < row_bytes; off += r.stage_bytes) {
        const uint32_t bytes = (uint32_t)umin64((uint64_t)r.stage_bytes, row_bytes - off);
        const uint32_t main_bytes = bytes & ~15u;
        const uint32_t s = q.s, ph = q.ph;
        mbar_wait(&r.full[s], ph);
        const uint8_t* sb = r.buf + s * r.stage_bytes;
        const uint32_t nvec = main_bytes / 16;
        // two 16-byte vectors per step: one max test per 2 VEC logits, four independent sums
        auto step = [&](uint32_t v, auto nv_tag) {
          constexpr int NV = decltype(nv_tag)::value;
          float z[VEC * NV];
#pragma unroll
          for (int u = 0; u < NV; ++u) RowVec<DT>::f32(lds128(sb + (v + u * kGT) * 16), z + VEC * u);
          float lm = z[0];
#pragma unroll
          for (int e = 1; e < VEC * NV; ++e) lm = fmaxf(lm, z[e]);
          if (lm > mz) {
            const float f = ex2_approx((mz - lm) * c);
            sum *= f;
            sum2 *= f;
            sum3 *= f;
            sum4 *= f;
            mz = lm;
            nb = -mz * c;
          }
#pragma unroll
          for (int e = 0; e < VEC * NV; e += 4) {
            sum += ex2_approx(fmaf(z[e], c, nb));
            sum2 += ex2_approx(fmaf(z[e + 1], c, nb));
            sum3 += ex2_approx(fmaf(z[e + 2], c, nb));
            sum4 += ex2_approx(fmaf(z[e + 3], c, nb));
          }
        };
        uint32_t v = tid;
        for (; v + kGT < nvec; v += 2 * kGT) step(v, std::integral_constant<int, 2>());
        if (v < nvec) step(v, std::integral_constant<int, 1>());
        for (uint32_t e = main_bytes / ESZ + tid; e < bytes / ESZ; e += kGT)
          take((float)load_f64<DT>(rowp, off / ESZ + e));
        __syncwarp();
        if (lane == 0) mbar_arrive(&r.empty[s]);
        q.next(r.nstages);
      }
    }
    sum = (sum + sum2) + (sum3 + sum4);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, mz, o), os = __shfl_xor_sync(0xffffffffu, sum, o);
      const float M = fmaxf(mz, om);
      sum = (M == -INFINITY) ? 0.f : sum * ex2_approx((mz - M) * c) + os * ex2_approx((om - M) * c);
      mz = M;
    }
    if (lane == 0) {
      ws[(row * kGW + warp) * 2] = mz;
      ws[(row * kGW + warp) * 2 + 1] = sum;
    }
  }
}

template <int DT>
__global__ void k_grpo_fwd_epilogue(FwdArgs a, const float* __restrict__ ws) {
  constexpr int ESZ = Elem<DT>::size;
  for (uint64_t row = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; row < a.n_rows;
       row += (uint64_t)gridDim.x * blockDim.x) {
    if (a.use[a.sample[row]] == 0) {
      if (a.logp) a.logp[row] = 0.0;
      if (a.lse) a.lse[row] = 0.0;
      a.term[row] = 0.0;
      a.coef[row] = 0.0;
      continue;
    }
    const double T = a.temp[a.sample[row]];
    const float2* pw = reinterpret_cast<const float2*>(ws + row * kGW * 2);
    float2 pr[kGW];
#pragma unroll
    for (int w = 0; w < kGW; ++w) pr[w] = pw[w];
    double M = pr[0].x;
#pragma unroll
    for (int w = 1; w < kGW; ++w) M = fmax(M, (double)pr[w].x);
    double S = 0.0;
#pragma unroll
    for (int w = 0; w < kGW; ++w)
      S += pr[w].x == -INFINITY ? 0.0 : (double)pr[w].y * exp2(((double)pr[w].x - M) * (kLog2e / T));
    const double lse = (T == 1.0 ? M : M / T) + log(S);  // lse of z / T (toy_env.py:172-174)
    const uint64_t rr = a.row_index ? (uint64_t)a.row_index[row] : row;
    fwd_epilogue<DT>(a, row, a.logits + rr * a.row_stride * ESZ, lse);
  }
}

// ------------------------------------------------------------------ K5 backward
struct BwdArgs {
  const char* logits;
  uint64_t n_out_rows, vocab, row_stride;
  const int64_t* logits_row;
  const int64_t* row_tok_ptr;
  const int64_t* row_tok;
  const int32_t* tokens;
  const double* temp;
  const double* lse;
  const double* coef;
  char* grad;
  uint64_t grad_row_stride;
};

__device__ __forceinline__ void tok_range(const BwdArgs& a, uint64_t o, int64_t& k0, int64_t& k1) {
  if (a.row_tok_ptr) { k0 = a.row_tok_ptr[o]; k1 = a.row_tok_ptr[o + 1]; }
  else { k0 = (int64_t)o; k1 = (int64_t)o + 1; }
}
__device__ __forceinline__ int64_t tok_at(const BwdArgs& a, int64_t k) { return a.row_tok ? a.row_tok[k] : k; }

template <int GT>
__device__ __forceinline__ void store_grad_f32(char* g, uint64_t idx, const float* v, int n) {
  if constexpr (GT == RLK_BF16) {
    if (n == 8) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        __nv_bfloat162 p = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
        w[e] = *reinterpret_cast<uint32_t*>(&p);
      }
      stg128_stream((uint16_t*)g + idx, make_uint4(w[0], w[1], w[2], w[3]));
    } else {
      for (int e = 0; e < n; ++e) reinterpret_cast<uint16_t*>(g)[idx + e] = f32_to_bf16_rne(v[e]);
    }
  } else if constexpr (GT == RLK_F32) {
    if (n % 4 == 0) {
      for (int e = 0; e < n; e += 4)
        stg128_stream((float*)g + idx + e, make_uint4(__float_as_uint(v[e]), __float_as_uint(v[e + 1]),
                                                       __float_as_uint(v[e + 2]), __float_as_uint(v[e + 3])));
    } else {
      for (int e = 0; e < n; ++e) reinterpret_cast<float*>(g)[idx + e] = v[e];
    }
  } else {
    for (int e = 0; e < n; ++e) reinterpret_cast<double*>(g)[idx + e] = (double)v[e];
  }
}

template <int DT, int GT>
__global__ void __launch_bounds__(kGThreads, 1) k_grpo_bwd(BwdArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int ESZ = Elem<DT>::size;
  constexpr int GSZ = Elem<GT>::size;
  constexpr int VEC = 16 / ESZ;
  constexpr bool F64MATH = (DT == RLK_F64) || (GT == RLK_F64);
  const Ring r = ring_setup(smem, kRowStageBytes, kRowStages, kGW);
  const uint64_t row_bytes = a.vocab * ESZ;
  auto lrow = [&](uint64_t o) { return a.logits_row ? (uint64_t)a.logits_row[o] : o; };
  auto active = [&](uint64_t o) {
    int64_t k0, k1;
    tok_range(a, o, k0, k1);
    for (int64_t k = k0; k < k1; ++k)
      if (a.coef[tok_at(a, k)] != 0.0) return true;
    return false;
  };
  auto addr = [&](uint64_t o) { return a.logits + lrow(o) * a.row_stride * ESZ; };
  auto streamed = [&](uint64_t o) { return active(o) && ((uintptr_t)addr(o) & 15u) == 0; };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  if (warp == kGW) {
    if (lane == 0) produce_rows(r, a.n_out_rows, row_bytes, streamed, addr);
    return;
  }
  RingPos q;
  for (uint64_t o = blockIdx.x; o < a.n_out_rows; o += gridDim.x) {
    char* grow = a.grad + lrow(o) * a.grad_row_stride * GSZ;
    if (!active(o)) {
      // objective.py:275-276 leaves the row at zero
      const uint64_t gbytes = a.vocab * GSZ;
      if (((uintptr_t)grow & 15u) == 0) {
        for (uint64_t b = (uint64_t)tid * 16; b + 16 <= gbytes; b += kGT * 16)
          stg128_stream(grow + b, make_uint4(0, 0, 0, 0));
        for (uint64_t b = (gbytes & ~15ull) + tid; b < gbytes; b += kGT) grow[b] = 0;
      } else {
        for (uint64_t b = tid; b < gbytes; b += kGT) grow[b] = 0;
      }
      continue;
    }
    int64_t k0, k1;
    tok_range(a, o, k0, k1);
    const char* rowp = addr(o);
    float rc_cf = 0.f, rc_c = 0.f, rc_nl = 0.f;
    int64_t rc_tok = -1;
    if (!F64MATH && a.row_tok_ptr == nullptr) {
      const double T = a.temp[o];
      rc_cf = (float)a.coef[o];
      rc_c = (float)(kLog2e / T);
      rc_nl = (float)(-a.lse[o] * kLog2e);
      rc_tok = a.tokens[o];
    }
    if (((uintptr_t)rowp & 15u) != 0 || ((uintptr_t)grow & 15u) != 0) {
      // unaligned row: reference-order f64 evaluation straight from global memory
      for (uint64_t v = tid; v < a.vocab; v += kGT) {
        const double z = load_f64<DT>(rowp, v);
        double g = 0.0;
        for (int64_t k = k0; k < k1; ++k) {
          const int64_t t = tok_at(a, k);
          const double cf = a.coef[t];
          if (cf == 0.0) continue;
          const double T = a.temp[t];
          const double p = exp(__dsub_rn(T == 1.0 ? z : __ddiv_rn(z, T), a.lse[t]));
          g = __dsub_rn(g, __dmul_rn(cf, p));
          if ((int64_t)v == (int64_t)a.tokens[t]) g = __dadd_rn(g, cf);
        }
        store_from_f64<GT>(grow, v, g);
      }
      continue;
    }
    for (uint64_t off = 0; off < row_bytes; off += r.stage_bytes) {
      const uint32_t bytes = (uint32_t)umin64((uint64_t)r.stage_bytes, row_bytes - off);
      const uint32_t main_bytes = bytes & ~15u;
      const uint32_t s = q.s, ph = q.ph;
      mbar_wait(&r.full[s], ph);
      const uint8_t* sb = r.buf + s * r.stage_bytes;
      const uint64_t v0 = off / ESZ;  // first vocab index of this stage
      const uint32_t nvec = main_bytes / 16;
      for (uint32_t v = tid; v < nvec + ((bytes - main_bytes) ? 1u : 0u); v += kGT) {
        const bool tail = v >= nvec;
        const int n = tail ? (int)((bytes - main_bytes) / ESZ) : VEC;
        const uint64_t vb = v0 + (uint64_t)v * VEC;
        if constexpr (F64MATH) {
          double z[VEC], g[VEC];
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            z[e] = 0.0;
            g[e] = 0.0;
          }
          if (!tail) {
            if constexpr (DT == RLK_F64) RowVec<RLK_F64>::f64(lds128(sb + v * 16), z);
            else {
              float zf[VEC];
              RowVec<DT>::f32(lds128(sb + v * 16), zf);
#pragma unroll
              for (int e = 0; e < VEC; ++e) z[e] = zf[e];
            }
          } else {
            for (int e = 0; e < n; ++e) z[e] = load_f64<DT>(rowp, vb + e);
          }
          for (int64_t k = k0; k < k1; ++k) {
            const int64_t t = tok_at(a, k);
            const double cf = a.coef[t];
            if (cf == 0.0) continue;
            const double T = a.temp[t], L = a.lse[t];
            const int64_t tk = a.tokens[t];
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              const double zt = T == 1.0 ? z[e] : __ddiv_rn(z[e], T);
              const double p = exp(__dsub_rn(zt, L));
              g[e] = __dsub_rn(g[e], __dmul_rn(cf, p));
              if ((int64_t)(vb + e) == tk) g[e] = __dadd_rn(g[e], cf);
            }
          }
          for (int e = 0; e < n; ++e) store_from_f64<GT>(grow, vb + e, g[e]);
        } else if (a.row_tok_ptr == nullptr) {
          // one token per row (the LM layout): row constants in registers, one-hot patched once
          float z[VEC], g[VEC];
          if (!tail) RowVec<DT>::f32(lds128(sb + v * 16), z);
          else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) z[e] = e < n ? (float)load_f64<DT>(rowp, vb + e) : 0.f;
          }
#pragma unroll
          for (int e = 0; e < VEC; e += 2) {
            g[e] = -rc_cf * ex2_approx(fmaf(z[e], rc_c, rc_nl));
            g[e + 1] = -rc_cf * ex2_approx(fmaf(z[e + 1], rc_c, rc_nl));
          }
          const int64_t rel = rc_tok - (int64_t)vb;
          if (rel >= 0 && rel < VEC) {
#pragma unroll
            for (int e = 0; e < VEC; ++e)
              if (e == rel) g[e] += rc_cf;
          }
          store_grad_f32<GT>(grow, vb, g, n);
        } else {
          float z[VEC], g[VEC];
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            z[e] = 0.f;
            g[e] = 0.f;
          }
          if (!tail) RowVec<DT>::f32(lds128(sb + v * 16), z);
          else
            for (int e = 0; e < n; ++e) z[e] = (float)load_f64<DT>(rowp, vb + e);
          for (int64_t k = k0; k < k1; ++k) {
            const int64_t t = tok_at(a, k);
            const double cfd = a.coef[t];
            if (cfd == 0.0) continue;
            const double T = a.temp[t];
            const float c = (float)(kLog2e / T), nl = (float)(-a.lse[t] * kLog2e), cf = (float)cfd;
            const int64_t tk = a.tokens[t];
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              g[e] = fmaf(-cf, ex2_approx(fmaf(z[e], c, nl)), g[e]);
              if ((int64_t)(vb + e) == tk) g[e] += cf;
            }
          }
          store_grad_f32<GT>(grow, vb, g, n);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&r.empty[s]);
      q.next(r.nstages);
    }
  }
}

// ------------------------------------------------------------------ log_token_dist rows (f64 math)
template <int DT, int OT>
__global__ void k_logsoftmax_rows(const char* logits, uint64_t n_rows, uint64_t vocab, uint64_t row_stride,
                                  const int64_t* row_index, const double* temp, char* out) {
  constexpr int ESZ = Elem<DT>::size;
  __shared__ double red_m[32], red_s[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (uint64_t row = blockIdx.x; row < n_rows; row += gridDim.x) {
    const uint64_t rr = row_index ? (uint64_t)row_index[row] : row;
    const char* rowp = logits + rr * row_stride * ESZ;
    const double T = temp[row];
    double m = -INFINITY;
    for (uint64_t v = threadIdx.x; v < vocab; v += blockDim.x) {
      const double z = load_f64<DT>(rowp, v);
      m = fmax(m, T == 1.0 ? z : __ddiv_rn(z, T));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red_m[warp] = m;
    __syncthreads();
    double M = red_m[0];
    for (int w = 1; w < nw; ++w) M = fmax(M, red_m[w]);
    double s = 0.0;
    for (uint64_t v = threadIdx.x; v < vocab; v += blockDim.x) {
      const double z = load_f64<DT>(rowp, v);
      s += exp(__dsub_rn(T == 1.0 ? z : __ddiv_rn(z, T), M));
    }
    s = warp_sum_f64(s);
    if (lane == 0) red_s[warp] = s;
    __syncthreads();
    double S = 0.0;
    for (int w = 0; w < nw; ++w) S += red_s[w];
    const double lse = M + log(S);  // toy_env.py:172-174
    for (uint64_t v = threadIdx.x; v < vocab; v += blockDim.x) {
      const double z = load_f64<DT>(rowp, v);
      store_from_f64<OT>(out, row * vocab + v, __dsub_rn(T == 1.0 ? z : __ddiv_rn(z, T), lse));
    }
    __syncthreads();
  }
}

// One 256-thread block per segment: thread t sums elements t, t + 256, ... of the segment, then a
// fixed shuffle / shared-memory tree -- the result depends only on the data, never on timing.
__global__ void k_segment_sum(const double* __restrict__ x, const int64_t* __restrict__ seg, uint64_t n_segs,
                              double* __restrict__ out) {
  __shared__ double red[8];
  for (uint64_t g = blockIdx.x; g < n_segs; g += gridDim.x) {
    double acc = 0.0;
    for (int64_t i = seg[g] + threadIdx.x; i < seg[g + 1]; i += blockDim.x) acc += x[i];
    acc = warp_sum_f64(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int w = 1; w < 8; ++w) t += red[w];
      out[g] = t;
    }
    __syncthreads();
  }
}

static int grid_rows(uint64_t n_rows) {
  const uint64_t sms = (uint64_t)sm_count();
  return (int)(n_rows < sms ? n_rows : sms);
}

template <typename K>
static int set_smem(K kern, uint32_t bytes) {
  return cuda_status(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
                     "cudaFuncSetAttribute");
}

template <int DT>
static int launch_fwd_split(const FwdArgs& a, float* ws, cudaStream_t s) {
  const uint32_t smem = 1024 + kRowStageBytes * (kRowStages / kK4aCtas);
  auto kern = k_grpo_fwd_stream<DT>;
  if (int st = set_smem(kern, smem)) return st;
  const uint64_t ctas = (uint64_t)sm_count() * kK4aCtas;
  kern<<<(unsigned)(a.n_rows < ctas ? a.n_rows : ctas), kGThreads, smem, s>>>(a, ws);
  if (int st = launch_status("rlk_grpo_fwd (stream)")) return st;
  const uint64_t blocks = (a.n_rows + 255) / 256;
  k_grpo_fwd_epilogue<DT><<<(unsigned)std::min<uint64_t>(blocks, 65535u * 16), 256, 0, s>>>(a, ws);
  return launch_status("rlk_grpo_fwd (epilogue)");
}

template <int DT>
static int launch_fwd(const FwdArgs& a, cudaStream_t s) {
  const uint32_t smem = 1024 + kRowStageBytes * kRowStages;
  auto kern = k_grpo_fwd<DT>;
  if (int st = set_smem(kern, smem)) return st;
  kern<<<grid_rows(a.n_rows), kGThreads, smem, s>>>(a);
  return launch_status("rlk_grpo_fwd");
}

template <int DT, int GT>
static int launch_bwd(const BwdArgs& a, cudaStream_t s) {
  const uint32_t smem = 1024 + kRowStageBytes * kRowStages;
  auto kern = k_grpo_bwd<DT, GT>;
  if (int st = set_smem(kern, smem)) return st;
  kern<<<grid_rows(a.n_out_rows), kGThreads, smem, s>>>(a);
  return launch_status("rlk_grpo_bwd");
}

template <int DT>
static int dispatch_bwd(int gt, const BwdArgs& a, cudaStream_t s) {
  switch (gt) {
    case RLK_BF16: return launch_bwd<DT, RLK_BF16>(a, s);
    case RLK_F32: return launch_bwd<DT, RLK_F32>(a, s);
    case RLK_F64: return launch_bwd<DT, RLK_F64>(a, s);
  }
  set_error("rlk_grpo_bwd: bad grad dtype %d", gt);
  return RLK_ERR_INVALID;
}

template <int DT>
static int dispatch_lsm(int ot, const char* lg, uint64_t n, uint64_t V, uint64_t st, const int64_t* ri,
                        const double* T, char* out, cudaStream_t s) {
  const int grid = grid_rows(n) * 4;
  switch (ot) {
    case RLK_BF16: k_logsoftmax_rows<DT, RLK_BF16><<<grid, 256, 0, s>>>(lg, n, V, st, ri, T, out); break;
    case RLK_F32: k_logsoftmax_rows<DT, RLK_F32><<<grid, 256, 0, s>>>(lg, n, V, st, ri, T, out); break;
    case RLK_F64: k_logsoftmax_rows<DT, RLK_F64><<<grid, 256, 0, s>>>(lg, n, V, st, ri, T, out); break;
    default: set_error("rlk_logsoftmax_rows: bad out dtype %d", ot); return RLK_ERR_INVALID;
  }
  return launch_status("rlk_logsoftmax_rows");
}


}  // namespace rlk

using namespace rlk;

extern "C" {

int rlk_grpo_fwd(const void* logits, int dtype, uint64_t n_rows, uint64_t vocab, uint64_t row_stride,
                 const int64_t* row_index, const int32_t* tokens, const double* logp_train, const double* logp_infer,
                 const int32_t* sample_of_row, const double* adv, const uint8_t* use, const double* temperature,
                 const double* norm, const rlk_clip* clip, double* logp_out, double* lse_out, double* term,
                 double* coef, int32_t* flags, float* workspace, uint64_t workspace_floats, void* stream) {
  if (n_rows == 0) return RLK_OK;
  RLK_REQUIRE(logits && tokens && logp_train && logp_infer && sample_of_row && adv && use && temperature && norm &&
                  clip && term && coef && flags,
              "rlk_grpo_fwd: NULL argument");
  RLK_REQUIRE(vocab >= 1 && row_stride >= vocab, "rlk_grpo_fwd: bad vocab/row_stride");
  RLK_REQUIRE(dtype >= RLK_BF16 && dtype <= RLK_F64, "rlk_grpo_fwd: bad dtype %d", dtype);
  const int esz = dtype == RLK_BF16 ? 2 : (dtype == RLK_F32 ? 4 : 8);
  RLK_REQUIRE(((uintptr_t)logits % esz) == 0, "rlk_grpo_fwd: logits must be element-aligned");
  FwdArgs a;
  a.logits = (const char*)logits;
  a.n_rows = n_rows;
  a.vocab = vocab;
  a.row_stride = row_stride;
  a.row_index = row_index;
  a.tokens = tokens;
  a.lp_train = logp_train;
  a.lp_infer = logp_infer;
  a.sample = sample_of_row;
  a.adv = adv;
  a.use = use;
  a.temp = temperature;
  a.norm = norm;
  a.clip = *clip;
  a.logp = logp_out;
  a.lse = lse_out;
  a.term = term;
  a.coef = coef;
  a.flags = flags;
  cudaStream_t s = (cudaStream_t)stream;
  const bool split = workspace && workspace_floats >= n_rows * 2 * (uint64_t)kGW && dtype != RLK_F64;
  switch (dtype) {
    case RLK_BF16: return split ? launch_fwd_split<RLK_BF16>(a, workspace, s) : launch_fwd<RLK_BF16>(a, s);
    case RLK_F32: return split ? launch_fwd_split<RLK_F32>(a, workspace, s) : launch_fwd<RLK_F32>(a, s);
    default: return launch_fwd<RLK_F64>(a, s);
  }
}

int rlk_segment_sum_f64(const double* x, const int64_t* seg_ptr, uint64_t n_segs, double* out, void* stream) {
  if (n_segs == 0) return RLK_OK;
  RLK_REQUIRE(x && seg_ptr && out, "rlk_segment_sum_f64: NULL argument");
  const unsigned grid = (unsigned)std::min<uint64_t>(n_segs, 65535u);
  k_segment_sum<<<grid, 256, 0, (cudaStream_t)stream>>>(x, seg_ptr, n_segs, out);
  return launch_status("rlk_segment_sum_f64");
}

int rlk_grpo_bwd(const void* logits, int dtype, uint64_t n_out_rows, uint64_t vocab, uint64_t row_stride,
                 const int64_t* logits_row, const int64_t* row_tok_ptr, const int64_t* row_tok, const int32_t* tokens,
                 const double* temperature_tok, const double* lse, const double* coef, void* grad, int grad_dtype,
                 uint64_t grad_row_stride, void* stream) {
  if (n_out_rows == 0) return RLK_OK;
  RLK_REQUIRE(logits && tokens && temperature_tok && lse && coef && grad, "rlk_grpo_bwd: NULL argument");
  RLK_REQUIRE(vocab >= 1 && row_stride >= vocab && grad_row_stride >= vocab, "rlk_grpo_bwd: bad strides");
  RLK_REQUIRE(dtype >= RLK_BF16 && dtype <= RLK_F64, "rlk_grpo_bwd: bad dtype %d", dtype);
  const int esz = dtype == RLK_BF16 ? 2 : (dtype == RLK_F32 ? 4 : 8);
  const int gsz = grad_dtype == RLK_BF16 ? 2 : (grad_dtype == RLK_F32 ? 4 : 8);
  RLK_REQUIRE(((uintptr_t)logits % esz) == 0 && ((uintptr_t)grad % gsz) == 0,
              "rlk_grpo_bwd: logits / grad must be element-aligned");
  BwdArgs a;
  a.logits = (const char*)logits;
  a.n_out_rows = n_out_rows;
  a.vocab = vocab;
  a.row_stride = row_stride;
  a.logits_row = logits_row;
  a.row_tok_ptr = row_tok_ptr;
  a.row_tok = row_tok;
  a.tokens = tokens;
  a.temp = temperature_tok;
  a.lse = lse;
  a.coef = coef;
  a.grad = (char*)grad;
  a.grad_row_stride = grad_row_stride;
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case RLK_BF16: return dispatch_bwd<RLK_BF16>(grad_dtype, a, s);
    case RLK_F32: return dispatch_bwd<RLK_F32>(grad_dtype, a, s);
    default: return dispatch_bwd<RLK_F64>(grad_dtype, a, s);
  }
}

int rlk_logsoftmax_rows(const void* logits, int dtype, uint64_t n_rows, uint64_t vocab, uint64_t row_stride,
                        const int64_t* row_index, const double* temperature_row, void* out, int out_dtype,
                        void* stream) {
  if (n_rows == 0) return RLK_OK;
  RLK_REQUIRE(logits && temperature_row && out, "rlk_logsoftmax_rows: NULL argument");
  RLK_REQUIRE(vocab >= 1 && row_stride >= vocab, "rlk_logsoftmax_rows: bad vocab/row_stride");
  cudaStream_t s = (cudaStream_t)stream;
  const char* lg = (const char*)logits;
  switch (dtype) {
    case RLK_BF16: return dispatch_lsm<RLK_BF16>(out_dtype, lg, n_rows, vocab, row_stride, row_index, temperature_row, (char*)out, s);
    case RLK_F32: return dispatch_lsm<RLK_F32>(out_dtype, lg, n_rows, vocab, row_stride, row_index, temperature_row, (char*)out, s);
    case RLK_F64: return dispatch_lsm<RLK_F64>(out_dtype, lg, n_rows, vocab, row_stride, row_index, temperature_row, (char*)out, s);
  }
  set_error("rlk_logsoftmax_rows: bad dtype %d", dtype);
  return RLK_ERR_INVALID;
}

}  // extern "C"
