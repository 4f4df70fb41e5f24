// margin_kernels.cu — K1 relay_margin_rows and K4 relay_step_switch (sm_100a).
//
// One streaming pass over each logit row (§3.2): online max with a
// lazily raised exp reference, the softmax normaliser in fp32 (MUFU.EX2 via
// ex2.approx, FFMA2/FADD2 pairs), and the exact top-2 (value desc, index asc)
// with a CTA-shared threshold so that only vectors that can still enter the
// row's top-2 take the exact per-element path.
// HBM-bound: algorithmic bytes = vocab * sizeof(elem) per row; no tensor cores
// (this is a scan, not a contraction).
#include "relay_device.cuh"
#include "relay_internal.h"

namespace relay {

struct ThreadState {
  Top2 t;
  float g2;    // own skip guard: NaN until t.i2 holds a real index, then t.v2
  float mref;  // exp reference in the y = z*c domain (never above the row max)
  float acc[4];
};

__device__ __forceinline__ void state_init(ThreadState& st) {
  st.t = top2_empty();
  st.g2 = qnan();
  st.mref = -FLT_MAX;
#pragma unroll
  for (int k = 0; k < 4; k++) st.acc[k] = 0.0f;
}

__device__ __forceinline__ void rescale(ThreadState& st, float ymax) {
  if (ymax > st.mref + kSlack) {
    float r = ex2(st.mref - ymax);
#pragma unroll
    for (int k = 0; k < 4; k++) st.acc[k] *= r;
    st.mref = ymax;
  }
}

// Exact path for one element (head/tail of a misaligned range).
__device__ __forceinline__ void consume_scalar(float x, int j, ThreadState& st, float c) {
  top2_push(st.t, x, j);
  st.g2 = (st.t.i2 == INT_MAX) ? qnan() : st.t.v2;
  rescale(st, x * c);
  st.acc[0] += ex2(fmaf(x, c, -st.mref));
}

// One vector of VEC consecutive elements starting at index j0.
template <int VEC>
__device__ __forceinline__ void consume_vec(const float (&f)[VEC], int j0, ThreadState& st,
                                            float c, float theta, bool& slow) {
  float vmax = f[0];
#pragma unroll
  for (int k = 1; k < VEC; k++) vmax = fmaxf(vmax, f[k]);
  // A vector can change the row's top-2 only if it holds a value >= theta
  // (theta <= the row's 2nd-best value) and one that beats this thread's own
  // 2nd-best (indices only grow along a thread's walk).
  bool s = (vmax >= theta) && !(vmax <= st.g2);
  if (s) {
#pragma unroll
    for (int k = 0; k < VEC; k++) top2_push(st.t, f[k], j0 + k);
    st.g2 = (st.t.i2 == INT_MAX) ? qnan() : st.t.v2;
  }
  slow |= s;
  rescale(st, vmax * c);
  const float2 cc = make_float2(c, c);
  const float2 nm = make_float2(-st.mref, -st.mref);
#pragma unroll
  for (int k = 0; k < VEC; k += 2) {
    float2 y = __ffma2_rn(make_float2(f[k], f[k + 1]), cc, nm);
    float2 e = make_float2(ex2(y.x), ex2(y.y));
    const int a = ((k >> 1) & 1) * 2;
    float2 acc = __fadd2_rn(make_float2(st.acc[a], st.acc[a + 1]), e);
    st.acc[a] = acc.x;
    st.acc[a + 1] = acc.y;
  }
}

template <class E, int VB>
struct Vec;

template <class E>
struct Vec<E, 16> {
  using Raw = uint4;
  static constexpr int N = 16 / E::SZ;
  __device__ static __forceinline__ Raw load(const char* p) { return ldg_stream16(p); }
  __device__ static __forceinline__ void unpack(const Raw& r, float (&f)[N]) {
    if constexpr (E::SZ == 4) {
      f[0] = __uint_as_float(r.x); f[1] = __uint_as_float(r.y);
      f[2] = __uint_as_float(r.z); f[3] = __uint_as_float(r.w);
    } else {
      E::unpack2(r.x, f[0], f[1]); E::unpack2(r.y, f[2], f[3]);
      E::unpack2(r.z, f[4], f[5]); E::unpack2(r.w, f[6], f[7]);
    }
  }
};

template <class E>
struct Vec<E, 32> {
  using Raw = U8x32;
  static constexpr int N = 32 / E::SZ;
  __device__ static __forceinline__ Raw load(const char* p) { return ldg_stream32(p); }
  __device__ static __forceinline__ void unpack(const Raw& r, float (&f)[N]) {
    if constexpr (E::SZ == 4) {
#pragma unroll
      for (int k = 0; k < 8; k++) f[k] = __uint_as_float(r.w[k]);
    } else {
#pragma unroll
      for (int k = 0; k < 8; k++) E::unpack2(r.w[k], f[2 * k], f[2 * k + 1]);
    }
  }
};

// Stream elements [j0, j1) of one row through this CTA (all threads call).
template <class E, int VB, int THREADS, int U>
__device__ __forceinline__ void stream_range(const typename E::T* __restrict__ row, int j0, int j1,
                                             float c, ThreadState& st, int* s_theta) {
  using V = Vec<E, VB>;
  constexpr int VEC = V::N;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(row + j0);
  int head = static_cast<int>(((VB - (addr & (VB - 1))) & (VB - 1)) / E::SZ);
  if (head > j1 - j0) head = j1 - j0;
  if (tid < head) consume_scalar(E::load1(row + j0 + tid), j0 + tid, st, c);
  const int jb = j0 + head;
  const int nvec = (j1 - jb) / VEC;
  const char* vbase = reinterpret_cast<const char*>(row + jb);
  // main loop: warp-uniform bound so the vote below sees all 32 lanes
  int wv = tid - lane;
  for (; wv + 31 + (U - 1) * THREADS < nvec; wv += U * THREADS) {
    const int v = wv + lane;
    typename V::Raw raw[U];
#pragma unroll
    for (int u = 0; u < U; u++) raw[u] = V::load(vbase + static_cast<size_t>(v + u * THREADS) * VB);
    const float theta = unkey(*reinterpret_cast<volatile int*>(s_theta));
    bool slow = false;
#pragma unroll
    for (int u = 0; u < U; u++) {
      float f[VEC];
      V::unpack(raw[u], f);
      consume_vec<VEC>(f, jb + (v + u * THREADS) * VEC, st, c, theta, slow);
    }
    if (__any_sync(kFull, slow)) {
      // the warp's two best values bound the row's 2nd-best from below
      float a = st.t.v1, b = st.t.v2;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        float oa = __shfl_xor_sync(kFull, a, off);
        float ob = __shfl_xor_sync(kFull, b, off);
        b = fmaxf(fminf(a, oa), fmaxf(b, ob));
        a = fmaxf(a, oa);
      }
      if (lane == 0 && b > unkey(*reinterpret_cast<volatile int*>(s_theta))) atomicMax(s_theta, fkey(b));
    }
  }
  for (int v = wv + lane; v < nvec; v += THREADS) {
    typename V::Raw raw = V::load(vbase + static_cast<size_t>(v) * VB);
    const float theta = unkey(*reinterpret_cast<volatile int*>(s_theta));
    bool slow = false;
    float f[VEC];
    V::unpack(raw, f);
    consume_vec<VEC>(f, jb + v * VEC, st, c, theta, slow);
  }
  const int jt = jb + nvec * VEC;
  if (tid < j1 - jt) consume_scalar(E::load1(row + jt + tid), jt + tid, st, c);
}

__device__ __forceinline__ Partial thread_partial(const ThreadState& st) {
  return Partial{st.t, Norm{st.mref, (st.acc[0] + st.acc[1]) + (st.acc[2] + st.acc[3])}};
}

__device__ __forceinline__ Partial partial_empty() {
  return Partial{top2_empty(), Norm{-FLT_MAX, 0.0f}};
}

template <int THREADS>
__device__ __forceinline__ Partial block_reduce(Partial p, Partial* s_red) {
  constexpr int NW = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  p = warp_reduce_partial(p);
  if (lane == 0) s_red[warp] = p;
  __syncthreads();
  if (warp == 0) {
    p = lane < NW ? s_red[lane] : partial_empty();
    p = warp_reduce_partial(p);
  }
  return p;  // valid in thread 0
}

// ------------------------------------------------------------------- K1
template <class E, int VB, int THREADS, int U>
__global__ void __launch_bounds__(THREADS)
    margin_rows_kernel(const typename E::T* __restrict__ logits, long long n_rows, int vocab,
                       long long stride, float c, float iota, float* __restrict__ margin,
                       int* __restrict__ top1, int* __restrict__ top2, float* __restrict__ lse,
                       uint8_t* __restrict__ status) {
  __shared__ int s_theta;
  __shared__ Partial s_red[THREADS / 32];
  for (long long r = blockIdx.x; r < n_rows; r += gridDim.x) {
    if (threadIdx.x == 0) s_theta = fkey(-INFINITY);
    __syncthreads();
    ThreadState st;
    state_init(st);
    stream_range<E, VB, THREADS, U>(logits + r * stride, 0, vocab, c, st, &s_theta);
    Partial p = block_reduce<THREADS>(thread_partial(st), s_red);
    if (threadIdx.x == 0) {
      RowOut o = finish_row(p, c, iota);
      margin[r] = o.margin;
      if (top1) top1[r] = o.i1;
      if (top2) top2[r] = o.i2;
      if (lse) lse[r] = o.lse;
      if (status) status[r] = static_cast<uint8_t>(o.status);
    }
    __syncthreads();
  }
}

static int g_num_sms = 0;

static int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <class E, int VB, int THREADS, int U>
static cudaError_t launch_rows_t(const void* logits, long long n_rows, int vocab, long long stride,
                                 float iota, float* margin, int* top1, int* top2, float* lse,
                                 uint8_t* status, cudaStream_t st) {
  auto kern = margin_rows_kernel<E, VB, THREADS, U>;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  long long grid = static_cast<long long>(per_sm) * num_sms();
  if (grid > n_rows) grid = n_rows;
  kern<<<static_cast<unsigned>(grid), THREADS, 0, st>>>(
      static_cast<const typename E::T*>(logits), n_rows, vocab, stride, iota * kLog2e, iota,
      margin, top1, top2, lse, status);
  return cudaGetLastError();
}

constexpr int kRowThreads = 512;

cudaError_t launch_margin_rows(const void* logits, int dt, long long n_rows, int vocab,
                               long long stride, float iota, float* margin, int* top1, int* top2,
                               float* lse, uint8_t* status, cudaStream_t st) {
  if (n_rows <= 0) return cudaSuccess;
  switch (dt) {
    case 0:
      return launch_rows_t<EBf16, 16, kRowThreads, 4>(logits, n_rows, vocab, stride, iota, margin,
                                                      top1, top2, lse, status, st);
    case 1:
      return launch_rows_t<EF16, 16, kRowThreads, 4>(logits, n_rows, vocab, stride, iota, margin,
                                                     top1, top2, lse, status, st);
    default:
      return launch_rows_t<EF32, 16, kRowThreads, 4>(logits, n_rows, vocab, stride, iota, margin,
                                                     top1, top2, lse, status, st);
  }
}

// ------------------------------------------------------------------- K4
// Runtime switching (§4.3, fig:mechanism P:209-216), one thread.
__device__ void switch_one(const CueDev& cs, int tok, float m, uint8_t* state_p, int* hist,
                           int* small_run_p, float gate, int max_seg, uint8_t* flag_out,
                           int16_t* cue_out) {
  int cue = -1, flag = 0;
  uint8_t state = *state_p;
  if (tok >= 0 && tok < cs.vocab && !(state & 2)) {
    int sr = small_run_p ? *small_run_p : 0;
    bool clear = false;
    if (tok == cs.think_end) {
      flag = 3; state = 3; clear = true;
    } else if ((state & 1) == 0) {
      int seq[kMaxLen];
#pragma unroll
      for (int k = 0; k < kHist; k++) seq[k] = hist[k];
      seq[kHist] = tok;
      int best = -1;
      for (int p = 0; p < cs.n_pat && best < 0; p++) {  // sorted by length desc
        const int len = cs.pat_len[p];
        bool ok = true;
        for (int k = 0; k < len; k++)
          if (seq[kMaxLen - len + k] != cs.pat_tok[p * kMaxLen + k]) { ok = false; break; }
        if (ok) best = p;
      }
      if (best >= 0 && !(gate >= 0.0f && m < gate)) {
        flag = 1; cue = cs.pat_cue[best]; state = 1; clear = true;
      } else {
        for (int k = 0; k < kHist - 1; k++) hist[k] = hist[k + 1];
        hist[kHist - 1] = tok;
      }
    } else {
      const bool term = (cs.term_tab[tok >> 5] >> (tok & 31)) & 1u;
      if (term) {
        flag = 2; state = 0; clear = true;
      } else if (max_seg > 0 && sr + 1 >= max_seg) {
        flag = 4; state = 0; clear = true;
      } else if (small_run_p) {
        *small_run_p = sr + 1;
      }
    }
    if (clear) {
      for (int k = 0; k < kHist; k++) hist[k] = -1;
      if (small_run_p) *small_run_p = 0;
    }
    *state_p = state;
  }
  *flag_out = static_cast<uint8_t>(flag);
  *cue_out = static_cast<int16_t>(cue);
}

template <class E, int VB, int THREADS, int U>
__global__ void __launch_bounds__(THREADS)
    step_switch_kernel(CueDev cs, const typename E::T* __restrict__ logits, int vocab,
                       long long stride, int nsplit, int chunk, float c, float iota,
                       const int* __restrict__ sampled, uint8_t* state, int* hist, int* small_run,
                       float gate, int max_seg, float* margin, int* top1, int* top2,
                       uint8_t* flag, int16_t* cue_id, int* counter, float* part) {
  __shared__ int s_theta;
  __shared__ Partial s_red[THREADS / 32];
  __shared__ int s_last;
  const int b = blockIdx.x / nsplit;
  const int k = blockIdx.x % nsplit;
  const int j0 = k * chunk;
  const int j1 = min(vocab, j0 + chunk);
  if (threadIdx.x == 0) s_theta = fkey(-INFINITY);
  __syncthreads();
  ThreadState st;
  state_init(st);
  if (j0 < j1) stream_range<E, VB, THREADS, U>(logits + b * stride, j0, j1, c, st, &s_theta);
  Partial p = block_reduce<THREADS>(thread_partial(st), s_red);
  if (threadIdx.x == 0) {
    float* q = part + (static_cast<size_t>(b) * nsplit + k) * 6;
    __stcg(q + 0, p.t.v1); __stcg(q + 1, p.t.v2);
    __stcg(q + 2, __int_as_float(p.t.i1)); __stcg(q + 3, __int_as_float(p.t.i2));
    __stcg(q + 4, p.n.m); __stcg(q + 5, p.n.s);
    __threadfence();
    const int old = atomicAdd(counter + b, 1);
    s_last = (old == nsplit - 1);
  }
  __syncthreads();
  if (!s_last) return;
  // last arriver for row b: merge the nsplit partials (one warp)
  __threadfence();
  if (threadIdx.x < 32) {
    Partial acc = partial_empty();
    for (int kk = threadIdx.x; kk < nsplit; kk += 32) {
      const float* q = part + (static_cast<size_t>(b) * nsplit + kk) * 6;
      Partial o;
      o.t.v1 = __ldcg(q + 0); o.t.v2 = __ldcg(q + 1);
      o.t.i1 = __float_as_int(__ldcg(q + 2)); o.t.i2 = __float_as_int(__ldcg(q + 3));
      o.n.m = __ldcg(q + 4); o.n.s = __ldcg(q + 5);
      acc = partial_merge(acc, o);
    }
    acc = warp_reduce_partial(acc);
    if (threadIdx.x == 0) {
      counter[b] = 0;  // ready for the next launch / graph replay
      RowOut o = finish_row(acc, c, iota);
      margin[b] = o.margin;
      if (top1) top1[b] = o.i1;
      if (top2) top2[b] = o.i2;
      const int tok = sampled ? sampled[b] : o.i1;
      switch_one(cs, tok, o.margin, state + b, hist + static_cast<size_t>(b) * kHist,
                 small_run ? small_run + b : nullptr, gate, max_seg, flag + b, cue_id + b);
    }
  }
}

constexpr int kStepThreads = 256;

template <class E>
static cudaError_t launch_step_t(const CueDev& cs, const void* logits, int batch, int vocab,
                                 long long stride, float iota, const int* sampled, uint8_t* state,
                                 int* hist, int* small_run, float gate, int max_seg, float* margin,
                                 int* top1, int* top2, uint8_t* flag, int16_t* cue_id,
                                 const StepWs& ws, cudaStream_t st) {
  // split rows so that the grid covers every SM several times
  int nsplit = (8 * num_sms() + batch - 1) / batch;
  if (nsplit > kMaxSplit) nsplit = kMaxSplit;
  if (nsplit < 1) nsplit = 1;
  int chunk = (vocab + nsplit - 1) / nsplit;
  chunk = (chunk + 63) / 64 * 64;
  if (chunk < 1024) chunk = 1024;
  nsplit = (vocab + chunk - 1) / chunk;
  auto kern = step_switch_kernel<E, 16, kStepThreads, 2>;
  kern<<<static_cast<unsigned>(batch) * nsplit, kStepThreads, 0, st>>>(
      cs, static_cast<const typename E::T*>(logits), vocab, stride, nsplit, chunk, iota * kLog2e,
      iota, sampled, state, hist, small_run, gate, max_seg, margin, top1, top2, flag, cue_id,
      ws.counter, ws.part);
  return cudaGetLastError();
}

cudaError_t launch_step_switch(const CueDev& cs, const void* logits, int dt, int batch, int vocab,
                               long long stride, float iota, const int* sampled, uint8_t* state,
                               int* hist, int* small_run, float gate, int max_seg, float* margin,
                               int* top1, int* top2, uint8_t* flag, int16_t* cue_id,
                               const StepWs& ws, cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  switch (dt) {
    case 0:
      return launch_step_t<EBf16>(cs, logits, batch, vocab, stride, iota, sampled, state, hist,
                                  small_run, gate, max_seg, margin, top1, top2, flag, cue_id, ws, st);
    case 1:
      return launch_step_t<EF16>(cs, logits, batch, vocab, stride, iota, sampled, state, hist,
                                 small_run, gate, max_seg, margin, top1, top2, flag, cue_id, ws, st);
    default:
      return launch_step_t<EF32>(cs, logits, batch, vocab, stride, iota, sampled, state, hist,
                                 small_run, gate, max_seg, margin, top1, top2, flag, cue_id, ws, st);
  }
}

}  // namespace relay
