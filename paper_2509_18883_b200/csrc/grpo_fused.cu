// Fused single-pass GRPO forward + backward (K4+K5 in one read of the logits): bf16 logits on 2-CTA
// clusters, f32 logits on 4-CTA clusters (each CTA owns V / cluster elements of the row: 128 KiB).
//
// objective_value and objective_gradient (pkg/src/rolloutlab/objective.py:230-283) both need the
// row's log-sum-exp; the backward additionally needs coef = norm * w * slope * r / T, known only after
// the whole row was reduced.  A row (V = 131072 bf16 = 256 KiB) does not fit one SM's shared memory,
// so a 2-CTA thread-block cluster owns it: each CTA streams its half into shared memory (TMA bulk
// copies, 16 KiB chunks, one mbarrier per chunk), reduces it (online max / sum of 2^(z c - m c)),
// and sends its (max, sum) partial into the peer CTA's shared memory with st.async, which completes
// a transaction on the peer's mbarrier -- no cluster-wide barrier per row.  Both CTAs then run the
// same f64 epilogue, write coef * (onehot - softmax) for their half from shared memory, and release
// each chunk to the producer, which is already streaming the next row in.  Logits are read once:
// 4 bytes of HBM traffic per logit for loss + gradient instead of 6 (K4 then K5).
#include "common.cuh"
#include "capi_internal.h"
#include "pipeline.cuh"

#include <type_traits>

namespace rlk {

constexpr int kFW = 16;                   // consumer warps
constexpr int kFT = kFW * 32;
constexpr int kFThreads = kFT + 64;       // + producer warp + epilogue warp
constexpr uint32_t kChunkBytes = 16384;   // TMA chunk (8192 bf16)
constexpr uint32_t kMaxHalfBytes = 200 * 1024;
constexpr double kLog2eF = 1.4426950408889634074;

__device__ __forceinline__ float ex2f_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t n_clusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
// 8-byte store into the peer CTA's shared memory, completing 8 tx bytes on the peer's mbarrier
__device__ __forceinline__ void st_async_peer(uint32_t remote_addr, float a, float b, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(remote_addr),
               "f"(a), "f"(b), "r"(remote_bar)
               : "memory");
}

struct FusedArgs {
  const char* logits;
  uint64_t n_rows, vocab, row_stride;
  const int64_t* row_index;
  const int32_t* tokens;
  const double *lp_train, *lp_infer;
  const int32_t* sample;
  const double* adv;
  const uint8_t* use;
  const double* temp;
  const double* norm;
  rlk_clip clip;
  double grad_scale;
  double *logp, *lse, *term, *coef;
  int32_t* flags;
  void* grad;
  uint64_t grad_row_stride;
  uint32_t nslots;
};

struct TripletF { double value, slope; };
__device__ __forceinline__ TripletF triplet_f(double r, double adv, const rlk_clip& c) {  // objective.py:133-150
  const double lo = 1.0 - c.eps_neg_low, hi = 1.0 + c.eps_pos_high;
  const double clipped = fmin(fmax(r, lo), hi);
  const double clip_slope = (lo <= r && r <= hi) ? 1.0 : 0.0;
  const double raw = __dmul_rn(r, adv), capped = __dmul_rn(clipped, adv);
  double inner, islope;
  if (raw <= capped) { inner = raw; islope = adv; }
  else { inner = capped; islope = __dmul_rn(adv, clip_slope); }
  if (c.guard_positive && adv > 0.0) return {inner, islope};
  const double floor_v = __dmul_rn(c.eps_neg_high, adv);
  if (inner >= floor_v) return {inner, islope};
  return {floor_v, 0.0};
}

__device__ __forceinline__ void unpack8(const uint4 w, float* z) {
  z[0] = bf16_lo(w.x); z[1] = bf16_hi(w.x); z[2] = bf16_lo(w.y); z[3] = bf16_hi(w.y);
  z[4] = bf16_lo(w.z); z[5] = bf16_hi(w.z); z[6] = bf16_lo(w.w); z[7] = bf16_hi(w.w);
}

// max of the bf16 pairs of two words, per half (max.bf16x2: HMNMX2.BF16, no unpacking)
__device__ __forceinline__ uint32_t hmax2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ float2 bf16x2_f32(uint32_t w) { return make_float2(bf16_lo(w), bf16_hi(w)); }

// Pass 1 over one chunk of a half row: online max / sum of 2^(z c - m c) in (mz, s[2] pairs); nb = -mz c.
// Two 16-byte vectors per thread per step (a full chunk is exactly two): one max test per 16 logits,
// the max taken on the packed bf16 words, the exponent arguments and sums in f32x2 (FFMA2 / FADD2).
struct RowAcc {
  float mz, nb;
  float2 s[2];
  __device__ void reset() {
    mz = -INFINITY;
    s[0] = s[1] = make_float2(0.f, 0.f);
    nb = INFINITY;
  }
  template <int NV>
  __device__ __forceinline__ void step(const uint8_t* cb, uint32_t v, float c) {
    uint32_t w[4 * NV];
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const uint4 q = lds128(cb + (v + u * kFT) * 16);
      w[4 * u] = q.x; w[4 * u + 1] = q.y; w[4 * u + 2] = q.z; w[4 * u + 3] = q.w;
    }
    uint32_t m2 = hmax2(w[0], w[1]);
#pragma unroll
    for (int k = 2; k < 4 * NV; ++k) m2 = hmax2(m2, w[k]);
    const float lm = fmaxf(bf16_lo(m2), bf16_hi(m2));
    if (lm > mz) rescale(lm, c);
#pragma unroll
    for (int k = 0; k < 4 * NV; ++k) {
      const float2 t = __ffma2_rn(bf16x2_f32(w[k]), make_float2(c, c), make_float2(nb, nb));
      s[k & 1] = __fadd2_rn(s[k & 1], make_float2(ex2f_approx(t.x), ex2f_approx(t.y)));
    }
  }
  // f32 logits: 4 values per 16-byte vector
  template <int NV>
  __device__ __forceinline__ void step_f32(const uint8_t* cb, uint32_t v, float c) {
    float z[4 * NV];
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const uint4 q = lds128(cb + (v + u * kFT) * 16);
      z[4 * u] = __uint_as_float(q.x); z[4 * u + 1] = __uint_as_float(q.y);
      z[4 * u + 2] = __uint_as_float(q.z); z[4 * u + 3] = __uint_as_float(q.w);
    }
    float lm = fmaxf(z[0], z[1]);
#pragma unroll
    for (int k = 2; k < 4 * NV; ++k) lm = fmaxf(lm, z[k]);
    if (lm > mz) rescale(lm, c);
#pragma unroll
    for (int k = 0; k < 2 * NV; ++k) {
      const float2 t = __ffma2_rn(make_float2(z[2 * k], z[2 * k + 1]), make_float2(c, c), make_float2(nb, nb));
      s[k & 1] = __fadd2_rn(s[k & 1], make_float2(ex2f_approx(t.x), ex2f_approx(t.y)));
    }
  }
  __device__ __forceinline__ void rescale(float lm, float c) {
    const float f = ex2f_approx((mz - lm) * c);
    s[0] = __fmul2_rn(s[0], make_float2(f, f));
    s[1] = __fmul2_rn(s[1], make_float2(f, f));
    mz = lm;
    nb = -mz * c;
  }
  template <int DT>
  __device__ __forceinline__ void chunk(const uint8_t* cb, uint32_t bytes, float c, int tid) {
    const uint32_t nv = bytes / 16;
    uint32_t v = tid;
    if constexpr (DT == RLK_BF16) {
      for (; v + kFT < nv; v += 2 * kFT) step<2>(cb, v, c);
      if (v < nv) step<1>(cb, v, c);
    } else {
      for (; v + kFT < nv; v += 2 * kFT) step_f32<2>(cb, v, c);
      if (v < nv) step_f32<1>(cb, v, c);
    }
  }
  __device__ __forceinline__ float sum() const { return (s[0].x + s[0].y) + (s[1].x + s[1].y); }
};

// Pass 2 over one chunk: grad = -cf * 2^(z c + nl) (the one-hot term is patched by the owner thread),
// exponent arguments and scaling in f32x2.
template <int NV>
__device__ __forceinline__ void grad_step(const uint8_t* cb, uint32_t v, float c, float ncf, float nl, uint16_t* gout) {
#pragma unroll
  for (int u = 0; u < NV; ++u) {
    RLK_DCHECK((v + u * kFT) * 16 < kChunkBytes);
    const uint4 q = lds128(cb + (v + u * kFT) * 16);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 t = __ffma2_rn(bf16x2_f32(w[e]), make_float2(c, c), make_float2(nl, nl));
      const float2 g = __fmul2_rn(make_float2(ex2f_approx(t.x), ex2f_approx(t.y)), make_float2(ncf, ncf));
      __nv_bfloat162 p2 = __floats2bfloat162_rn(g.x, g.y);
      o[e] = *reinterpret_cast<uint32_t*>(&p2);
    }
    stg128_stream(gout + (uint64_t)(v + u * kFT) * 8, make_uint4(o[0], o[1], o[2], o[3]));
  }
}

template <int NV>
__device__ __forceinline__ void grad_step_f32(const uint8_t* cb, uint32_t v, float c, float ncf, float nl, float* gout) {
#pragma unroll
  for (int u = 0; u < NV; ++u) {
    RLK_DCHECK((v + u * kFT) * 16 < kChunkBytes);
    const uint4 q = lds128(cb + (v + u * kFT) * 16);
    const float2 t0 = __ffma2_rn(make_float2(__uint_as_float(q.x), __uint_as_float(q.y)), make_float2(c, c),
                                 make_float2(nl, nl));
    const float2 t1 = __ffma2_rn(make_float2(__uint_as_float(q.z), __uint_as_float(q.w)), make_float2(c, c),
                                 make_float2(nl, nl));
    const float2 g0 = __fmul2_rn(make_float2(ex2f_approx(t0.x), ex2f_approx(t0.y)), make_float2(ncf, ncf));
    const float2 g1 = __fmul2_rn(make_float2(ex2f_approx(t1.x), ex2f_approx(t1.y)), make_float2(ncf, ncf));
    stg128_stream(gout + (uint64_t)(v + u * kFT) * 4, make_uint4(__float_as_uint(g0.x), __float_as_uint(g0.y),
                                                                 __float_as_uint(g1.x), __float_as_uint(g1.y)));
  }
}

// (M, S) of the lanes' (m, s) pairs: max and sum of s * 2^((m - M) c); empty pairs have m = -inf.
__device__ __forceinline__ void warp_combine(float& mz, float& sum, float c, unsigned mask = 0xffffffffu) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(mask, mz, o), os = __shfl_xor_sync(mask, sum, o);
    const float M = fmaxf(mz, om);
    sum = (M == -INFINITY) ? 0.f : sum * ex2f_approx((mz - M) * c) + os * ex2f_approx((om - M) * c);
    mz = M;
  }
}

// Per-row operands the consumers need, published in shared memory by the epilogue warp one row ahead
// (so the dependent global loads sample -> use / temperature never sit on the consumers' path).
struct RowInfo {
  uint64_t row;   // next active row (>= n_rows: none)
  uint64_t lrow;  // its logits / grad row (row_index)
  float c;        // log2(e) / temperature
  int32_t tok;    // target token
};
static_assert(896 + 2 * sizeof(RowInfo) <= 1024, "RowInfo must fit the 1 KiB header");

// Warp roles: 16 consumer warps (both passes), one producer warp (lane 0 issues TMA), one epilogue
// warp.  Rows are software-pipelined: after pass 1 of row r the consumers hand their partials to the
// epilogue warp (mbarrier), run pass 1 over the chunks of the next row that are already in the ring,
// and only then wait for row r's coefficient and run its pass 2 -- the cross-CTA exchange and the
// serial epilogue are off the consumers' critical path.
// DT: logits (and gradient) dtype; CL: CTAs per cluster = per row (set at launch).
template <int DT, int CL>
__global__ void __launch_bounds__(kFThreads, 1) k_grpo_fused(FusedArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // 1 KiB header: [full[nslots] | empty[nslots] | xbar[2] | pready[2] | cready[2] | ibar[2]] (<= 512 B),
  // slot[2][CL] float2 @512, bcast[2][4] float @576, red[2][kFW][2] float @640, info[2] RowInfo @896
  static_assert(2 * CL * 8 <= 64, "peer partial slots overflow the header");
  constexpr int ESZ = Elem<DT>::size;
  constexpr uint32_t kCE = kChunkBytes / ESZ;  // elements per chunk
  constexpr uint32_t kVE = 16 / ESZ;           // elements per 16-byte vector
  using GT = typename std::conditional<DT == RLK_BF16, uint16_t, float>::type;
  const uint32_t rank = cluster_rank();
  const uint64_t half = a.vocab / CL;  // elements owned by this CTA (vocab % (8 CL) == 0)
  const uint64_t v0 = rank * half;
  const uint32_t half_bytes = (uint32_t)(half * ESZ);
  const uint32_t nch = (half_bytes + kChunkBytes - 1) / kChunkBytes;  // chunks per half row
  const uint32_t nslots = a.nslots;  // ring slots >= nch: the producer runs ahead into the next row
  const uint32_t pre = min(nch, nslots - nch);  // next-row chunks that fit beside the current row
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + nslots;
  uint64_t* xbar = empty + nslots;
  uint64_t* pready = xbar + 2;
  uint64_t* cready = pready + 2;
  uint64_t* ibar = cready + 2;
  float2* slot = reinterpret_cast<float2*>(smem + 512);
  RowInfo* info = reinterpret_cast<RowInfo*>(smem + 896);
  float* bcast = reinterpret_cast<float*>(smem + 576);
  float* red = reinterpret_cast<float*>(smem + 640);
  uint8_t* buf = smem + 1024;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  if (threadIdx.x == 0) {
    for (uint32_t k = 0; k < nslots; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], kFW);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&xbar[k], 1);
      mbar_init(&pready[k], kFW);
      mbar_init(&cready[k], 1);
      mbar_init(&ibar[k], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  cluster_sync_all();  // peers' barriers exist before any st.async targets them

  auto active = [&](uint64_t row) { return a.use[a.sample[row]] != 0; };
  auto lrow = [&](uint64_t row) { return a.row_index ? (uint64_t)a.row_index[row] : row; };
  const uint64_t row0 = cluster_id_x(), rstep = n_clusters_x();

  if (warp == kFW) {
    // ---------------- producer: chunk k of every active row into the next ring slot
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      RingPos q;
      for (uint64_t row = row0; row < a.n_rows; row += rstep) {
        if (!active(row)) continue;
        const char* src = a.logits + (lrow(row) * a.row_stride + v0) * ESZ;
        for (uint32_t k = 0; k < nch; ++k) {
          const uint32_t bytes = min(kChunkBytes, half_bytes - k * kChunkBytes);
          RLK_DCHECK(q.s < nslots && bytes > 0 && (uint64_t)k * kChunkBytes + bytes <= half_bytes);
          mbar_wait(&empty[q.s], q.ph ^ 1u);
          mbar_arrive_expect_tx(&full[q.s], bytes);
          bulk_g2s(buf + q.s * kChunkBytes, src + (uint64_t)k * kChunkBytes, bytes, &full[q.s], pol);
          q.next(nslots);
        }
      }
    }
  } else if (warp == kFW + 1) {
    // ---------------- epilogue warp: combine partials, exchange with the peer, per-row outputs
    uint32_t ph[2] = {0u, 0u};
    uint64_t it = 0;
    for (uint64_t row = row0; row < a.n_rows; row += rstep) {
      if (!active(row)) continue;
      const uint32_t p = (uint32_t)(it++ & 1u);
      if (lane == 0) {
        // the consumers read this after pass 1 of `row` (ibar[p] completes once per use of parity p;
        // info[p] of two rows back was consumed before pass 2 of the previous row started)
        uint64_t nr = row + rstep;
        while (nr < a.n_rows && !active(nr)) nr += rstep;
        RowInfo ni;
        ni.row = nr;
        ni.lrow = 0;
        ni.c = 0.f;
        ni.tok = 0;
        if (nr < a.n_rows) {
          ni.lrow = lrow(nr);
          ni.c = (float)(kLog2eF / a.temp[a.sample[nr]]);
          ni.tok = a.tokens[nr];
        }
        info[p] = ni;
        mbar_arrive(&ibar[p]);
      }
      const int32_t s_id = a.sample[row];
      const double T = a.temp[s_id];
      const float c = (float)(kLog2eF / T);
      int32_t tok = 0;
      double zt = 0.0, lt64 = 0.0, li64 = 0.0, adv = 0.0, nrm = 0.0;
      if (lane == 0) {
        mbar_arrive_expect_tx(&xbar[p], 8 * (CL - 1));  // the peers' partials land in slot[p][r]
        tok = a.tokens[row];
        lt64 = a.lp_train[row];
        li64 = a.lp_infer[row];
        adv = a.adv[s_id];
        nrm = a.norm[s_id];
        if (tok >= 0 && (uint64_t)tok < a.vocab) zt = load_f64<DT>(a.logits + lrow(row) * a.row_stride * ESZ, (uint64_t)tok);
      }
      mbar_wait(&pready[p], ph[p]);
      float M = -INFINITY, S = 0.f;
      if (lane < kFW) {
        M = red[(p * kFW + lane) * 2];
        S = red[(p * kFW + lane) * 2 + 1];
      }
      warp_combine(M, S, c);
      if (lane == 0) {
        RLK_DCHECK(p < 2 && rank < (uint32_t)CL);
#pragma unroll
        for (uint32_t r = 0; r < (uint32_t)CL; ++r)
          if (r != rank) st_async_peer(mapa(smem_u32(&slot[p * CL + rank]), r), M, S, mapa(smem_u32(&xbar[p]), r));
        mbar_wait(&xbar[p], ph[p]);
        // combine and run the epilogue (objective.py:243-248, 277-279) in float64, like K4's: this
        // warp is off the consumers' critical path, so the precise exp / log cost nothing (an f32
        // epilogue loses ~1e-5 absolute in logp = z/T - lse when |z/T| reaches hundreds).
        // Every CTA combines the partials in rank order, so all compute the same numbers; rank 0
        // writes the per-token outputs.
        float2 part[CL];
#pragma unroll
        for (int r = 0; r < CL; ++r) part[r] = (uint32_t)r == rank ? make_float2(M, S) : slot[p * CL + r];
        float Mm = part[0].x;
#pragma unroll
        for (int r = 1; r < CL; ++r) Mm = fmaxf(Mm, part[r].x);
        double Sd = 0.0;
#pragma unroll
        for (int r = 0; r < CL; ++r)
          if (part[r].x != -INFINITY) Sd += (double)part[r].y * exp2(((double)part[r].x - (double)Mm) * (double)c);
        const double lse = (double)Mm / T + log(Sd);  // ln-sum-exp of z / T
        double cf = 0.0;
        if (tok < 0 || (uint64_t)tok >= a.vocab) {
          if (rank == 0) {
            atomicOr(a.flags, 2);
            if (a.logp) a.logp[row] = nan("");
            if (a.lse) a.lse[row] = lse;
            a.term[row] = 0.0;
            a.coef[row] = 0.0;
          }
        } else {
          const double logp = zt / T - lse;
          const double r = exp(logp - lt64);
          const double w = fmin(exp(lt64 - li64), a.clip.tis_cap);
          const TripletF tv = triplet_f(r, adv, a.clip);
          cf = nrm * w * tv.slope * r / T;
          if (rank == 0) {
            if (!isfinite(logp)) atomicOr(a.flags, 1);
            if (a.logp) a.logp[row] = logp;
            if (a.lse) a.lse[row] = lse;
            a.term[row] = w * tv.value;
            a.coef[row] = cf;
          }
        }
        bcast[p * 4 + 0] = (float)(cf * a.grad_scale);
        bcast[p * 4 + 1] = (float)(-lse * kLog2eF);
        mbar_arrive(&cready[p]);
      }
      ph[p] ^= 1u;
      __syncwarp();
    }
  } else {
    // ---------------- consumers
    uint32_t cph[2] = {0u, 0u};
    uint64_t it = 0;
    RingPos q;        // next ring position to wait on (pass 1)
    RowAcc acc;
    acc.reset();
    uint32_t done = 0;  // chunks of the current row already reduced by the previous iteration's pre-pass
    uint32_t iph[2] = {0u, 0u};
    // zero the gradient and outputs of inactive rows (objective.py:240-241 / 275-276)
    auto zero_row = [&](uint64_t row) {
      GT* grow = reinterpret_cast<GT*>(a.grad) + lrow(row) * a.grad_row_stride + v0;
      for (uint64_t b = (uint64_t)tid * kVE; b < half; b += (uint64_t)kFT * kVE)
        stg128_stream(grow + b, make_uint4(0, 0, 0, 0));
      if (rank == 0 && tid == 0) {
        if (a.logp) a.logp[row] = 0.0;
        if (a.lse) a.lse[row] = 0.0;
        a.term[row] = 0.0;
        a.coef[row] = 0.0;
      }
    };
    uint64_t row = row0;
    for (; row < a.n_rows && !active(row); row += rstep) zero_row(row);
    float c = 0.f;
    int32_t tok = 0;
    uint64_t lr = 0;
    if (row < a.n_rows) {
      c = (float)(kLog2eF / a.temp[a.sample[row]]);
      tok = a.tokens[row];
      lr = lrow(row);
    }
    RingPos q_row = q;  // ring position of the current row's chunk 0
    while (row < a.n_rows) {
      const uint32_t p = (uint32_t)(it++ & 1u);
      // pass 1 (rest of the row)
      for (uint32_t k = done; k < nch; ++k) {
        mbar_wait(&full[q.s], q.ph);
        acc.chunk<DT>(buf + q.s * kChunkBytes, min(kChunkBytes, half_bytes - k * kChunkBytes), c, tid);
        q.next(nslots);
      }
      float mz = acc.mz, sum = acc.sum();
      warp_combine(mz, sum, c);
      if (lane == 0) {
        red[(p * kFW + warp) * 2] = mz;
        red[(p * kFW + warp) * 2 + 1] = sum;
        mbar_arrive(&pready[p]);
      }
      // pass 1 of the next active row over the chunks already in the ring
      mbar_wait(&ibar[p], iph[p]);
      iph[p] ^= 1u;
      const RowInfo ni = info[p];
      const uint64_t nrow = ni.row;
      for (uint64_t zr = row + rstep; zr < nrow && zr < a.n_rows; zr += rstep) zero_row(zr);
      const RingPos q_next = q;
      acc.reset();
      done = 0;
      if (nrow < a.n_rows) {
        const float cn = ni.c;
        for (; done < pre; ++done) {
          mbar_wait(&full[q.s], q.ph);
          acc.chunk<DT>(buf + q.s * kChunkBytes, min(kChunkBytes, half_bytes - done * kChunkBytes), cn, tid);
          q.next(nslots);
        }
      }
      // pass 2 of this row: grad = cf * (onehot - 2^(z c - lse log2 e)), chunk by chunk
      mbar_wait(&cready[p], cph[p]);
      cph[p] ^= 1u;
      const float cf = bcast[p * 4 + 0], nl = bcast[p * 4 + 1];
      GT* grow = reinterpret_cast<GT*>(a.grad) + lr * a.grad_row_stride + v0;
      // the chunk / vector / thread that holds the target token's logit (the one-hot term)
      const int64_t tok_local = (int64_t)tok - (int64_t)v0;
      const bool tok_here = tok_local >= 0 && tok_local < (int64_t)half;
      const uint32_t tok_chunk = tok_here ? (uint32_t)(tok_local / kCE) : 0xffffffffu;
      const uint32_t tok_vec = tok_here ? (uint32_t)(tok_local % kCE) / kVE : 0u;
      RingPos q2 = q_row;
      for (uint32_t k = 0; k < nch; ++k) {
        const uint32_t bytes = min(kChunkBytes, half_bytes - k * kChunkBytes);
        const uint8_t* cb = buf + q2.s * kChunkBytes;
        GT* gout = grow + (uint64_t)k * kCE;
        const uint32_t nv = bytes / 16;
        if (cf == 0.f) {  // no gradient for this row (objective.py:277-279 with coef 0)
          for (uint32_t v = tid; v < nv; v += kFT) stg128_stream(gout + (uint64_t)v * kVE, make_uint4(0, 0, 0, 0));
        } else {
          uint32_t v = tid;
          if constexpr (DT == RLK_BF16) {
            for (; v + kFT < nv; v += 2 * kFT) grad_step<2>(cb, v, c, -cf, nl, gout);
            if (v < nv) grad_step<1>(cb, v, c, -cf, nl, gout);
          } else {
            for (; v + kFT < nv; v += 2 * kFT) grad_step_f32<2>(cb, v, c, -cf, nl, gout);
            if (v < nv) grad_step_f32<1>(cb, v, c, -cf, nl, gout);
          }
          if (k == tok_chunk && tok_vec % kFT == (uint32_t)tid) {
            // same thread, after its vector store: cf * (1 - softmax) at the target
            const uint32_t e = (uint32_t)(tok_local % kCE);
            float z;
            if constexpr (DT == RLK_BF16) z = __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(cb)[e] << 16);
            else z = reinterpret_cast<const float*>(cb)[e];
            const float g = cf - cf * ex2f_approx(fmaf(z, c, nl));
            if constexpr (DT == RLK_BF16) {
              __nv_bfloat16 hb = __float2bfloat16_rn(g);
              gout[e] = *reinterpret_cast<uint16_t*>(&hb);
            } else {
              gout[e] = g;
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[q2.s]);
        q2.next(nslots);
      }
      row = nrow;
      c = ni.c;
      tok = ni.tok;
      lr = ni.lrow;
      q_row = q_next;
    }
  }
  __syncwarp();
  cluster_sync_all();  // no CTA leaves while its peers may still st.async into it
}

}  // namespace rlk

using namespace rlk;

template <int DT, int CL>
static int launch_fused(const FusedArgs& a, uint32_t smem, cudaStream_t stream) {
  auto kern = k_grpo_fused<DT, CL>;
  if (int st = cuda_status(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                           "cudaFuncSetAttribute"))
    return st;
  if (int st = cuda_status(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                           "cudaFuncSetAttribute"))
    return st;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kFThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent clusters: exactly as many as can be co-resident (a cluster must fit in one GPC, so with
  // 4-CTA clusters some SMs stay idle -- launching sm_count / CL would leave a second wave of clusters
  // waiting for whole row sequences of the first)
  cfg.gridDim = dim3((unsigned)(CL * (sm_count() / CL)), 1, 1);
  int max_clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters <= 0) {
    cudaGetLastError();
    max_clusters = sm_count() / CL;
  }
  const uint64_t clusters = std::max<uint64_t>(1, std::min<uint64_t>(a.n_rows, (uint64_t)max_clusters));
  cfg.gridDim = dim3((unsigned)(CL * clusters), 1, 1);
  if (int st = cuda_status(cudaLaunchKernelEx(&cfg, kern, a), "cudaLaunchKernelEx")) return st;
  return launch_status("rlk_grpo_fused");
}

extern "C" int rlk_grpo_fused(const void* logits, int dtype, uint64_t n_rows, uint64_t vocab, uint64_t row_stride,
                              const int64_t* row_index, const int32_t* tokens, const double* logp_train,
                              const double* logp_infer, const int32_t* sample_of_row, const double* adv,
                              const uint8_t* use, const double* temperature, const double* norm, const rlk_clip* clip,
                              double grad_scale, double* logp_out, double* lse_out, double* term, double* coef,
                              int32_t* flags, void* grad, uint64_t grad_row_stride, void* stream) {
  if (n_rows == 0) return RLK_OK;
  RLK_REQUIRE(logits && tokens && logp_train && logp_infer && sample_of_row && adv && use && temperature && norm &&
                  clip && term && coef && flags && grad,
              "rlk_grpo_fused: NULL argument");
  RLK_REQUIRE(dtype == RLK_BF16 || dtype == RLK_F32, "rlk_grpo_fused: logits must be bf16 or f32 (got %d)", dtype);
  const int esz = dtype == RLK_BF16 ? 2 : 4;
  const int cl = dtype == RLK_BF16 ? 2 : 4;  // CTAs per row: each owns vocab * esz / cl bytes
  RLK_REQUIRE(vocab % (8 * cl) == 0 && vocab * esz / cl <= kMaxHalfBytes,
              "rlk_grpo_fused: vocab must be a multiple of %d and at most %u", 8 * cl, kMaxHalfBytes * cl / esz);
  RLK_REQUIRE(row_stride % (16 / esz) == 0 && grad_row_stride % (16 / esz) == 0 && ((uintptr_t)logits & 15u) == 0 &&
                  ((uintptr_t)grad & 15u) == 0,
              "rlk_grpo_fused: rows must be 16-byte aligned");
  FusedArgs a;
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
  a.grad_scale = grad_scale;
  a.logp = logp_out;
  a.lse = lse_out;
  a.term = term;
  a.coef = coef;
  a.flags = flags;
  a.grad = grad;
  a.grad_row_stride = grad_row_stride;
  const uint32_t part_bytes = (uint32_t)(vocab * esz / cl);
  const uint32_t nch = (part_bytes + kChunkBytes - 1) / kChunkBytes;
  a.nslots = std::max<uint32_t>(nch, std::min<uint32_t>(60u, (226u * 1024u - 1024u) / kChunkBytes));
  const uint32_t smem = 1024 + a.nslots * kChunkBytes;
  cudaStream_t s = (cudaStream_t)stream;
  return dtype == RLK_BF16 ? launch_fused<RLK_BF16, 2>(a, smem, s) : launch_fused<RLK_F32, 4>(a, smem, s);
}

extern "C" int rlk_grpo_fused_bf16(const void* logits, uint64_t n_rows, uint64_t vocab, uint64_t row_stride,
                                   const int64_t* row_index, const int32_t* tokens, const double* logp_train,
                                   const double* logp_infer, const int32_t* sample_of_row, const double* adv,
                                   const uint8_t* use, const double* temperature, const double* norm,
                                   const rlk_clip* clip, double grad_scale, double* logp_out, double* lse_out,
                                   double* term, double* coef, int32_t* flags, void* grad, uint64_t grad_row_stride,
                                   void* stream) {
  return rlk_grpo_fused(logits, RLK_BF16, n_rows, vocab, row_stride, row_index, tokens, logp_train, logp_infer,
                        sample_of_row, adv, use, temperature, norm, clip, grad_scale, logp_out, lse_out, term, coef,
                        flags, grad, grad_row_stride, stream);
}
