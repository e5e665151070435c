// K8r: deterministic replay of the reference's sequential per-worker epoch
// (optimizer.hpp:232-307) entirely on the device.
//
//  1. k_mt_words   — each worker's std::mt19937_64 stream (rng.hpp:42-84),
//                    one CTA per worker: the 312-word twist in two parallel
//                    halves, tempering, the epoch's (1 + s) words per draw.
//  2. k_replay_map — words -> head = eligible[uniform_index(|eligible|)],
//                    tails = pool[uniform_index(|pool|)] (optimizer.hpp:
//                    254-255, :284-285); a word in the rejection region of
//                    rng.hpp:49-55 (probability n / 2^64) flags the worker,
//                    whose epoch is then drawn on the host from the saved
//                    start state.
//  3. deps         — per draw its touch list (head, neighbours, tails,
//                    duplicates removed), per point the draws touching it in
//                    draw order (count, scan, scatter, per-point sort), and
//                    per (draw, point) the latest earlier draw touching it.
//  4. k_sgd_dataflow — persistent kernel; warps claim 32 consecutive draws of
//                    a worker in worker-interleaved order; a draw runs once
//                    every predecessor is done, so each point sees its updates
//                    in exactly the sequential order and positions are
//                    bit-identical (the arithmetic is the reference's op
//                    order with _rn intrinsics).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include <cub/cub.cuh>

#include "common.cuh"
#include "replay.cuh"
#include "sgd_device.cuh"

namespace nb {

// ---------------------------------------------------------- MT19937-64
constexpr unsigned long long kMtA = 0xB5026F5AA96619E9ull;
constexpr unsigned long long kMtUM = 0xFFFFFFFF80000000ull, kMtLM = 0x7FFFFFFFull;

__host__ __device__ __forceinline__ unsigned long long mt_temper(unsigned long long x) {
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}
// one step of the twist: (upper bit of a | lower 63 of b), shifted, xor A if odd
__host__ __device__ __forceinline__ unsigned long long mt_mix(unsigned long long a,
                                                              unsigned long long b) {
  const unsigned long long x = (a & kMtUM) | (b & kMtLM);
  return (x >> 1) ^ ((x & 1ull) ? kMtA : 0ull);
}

void Mt64::seed(uint64_t v) {
  s.mt[0] = v;
  for (uint32_t i = 1; i < 312; ++i)
    s.mt[i] = 6364136223846793005ull * (s.mt[i - 1] ^ (s.mt[i - 1] >> 62)) + i;
  s.p = 312;
  s.pad = 0;
}
void Mt64::twist() {
  for (uint32_t i = 0; i < 312; ++i)
    s.mt[i] = s.mt[(i + 156) % 312] ^ mt_mix(s.mt[i], s.mt[(i + 1) % 312]);
  s.p = 0;
}
uint64_t Mt64::next() {
  if (s.p >= 312) twist();
  return mt_temper(s.mt[s.p++]);
}

// One CTA per worker. Thread j < 156 of a twist owns words j and j + 156:
//   new[j]       = old[j + 156] ^ mix(old[j], old[j + 1])            (j < 156)
//   new[j + 156] = new[j] ^ mix(old[j + 156], old[j + 157] | new[0])  (j = 155: new[0])
// which is the standard's in-place sequential loop.
__global__ void __launch_bounds__(160) k_mt_words(ReplayDev R, const uint64_t* counts) {
  __shared__ unsigned long long s[312];
  const uint32_t w = blockIdx.x, tid = threadIdx.x;
  const MtState* in = R.st_in + w;
  for (uint32_t i = tid; i < 312; i += blockDim.x) s[i] = in->mt[i];
  uint32_t p = in->p;
  const uint64_t n = counts[w];
  unsigned long long* o = R.words + R.word_base[w];
  __syncthreads();
  uint64_t done = 0;
  {
    const uint64_t take = p < 312 ? std::min<uint64_t>(312 - p, n) : 0;
    for (uint32_t i = tid; i < take; i += blockDim.x) o[i] = mt_temper(s[p + i]);
    done = take;
    p += (uint32_t)take;
  }
  // One twist per 312 words (rng.hpp:42-84; Mt64::twist): thread t < 156
  // forms new[t] = old[t+156] ^ mix(old[t], old[t+1]) and new[t+156] =
  // new[t] ^ mix(old[t+156], old[t+157]) — the last one mixing with new[0],
  // which thread 155 forms itself from the old words — and writes both
  // tempered words from registers: two barriers per 312 words.
  while (done < n) {
    unsigned long long a0 = 0, a1 = 0, b0 = 0, b1 = 0;
    if (tid < 156) {
      a0 = s[tid];
      a1 = s[tid + 1];
      b0 = s[tid + 156];
      b1 = tid < 155 ? s[tid + 157] : s[156] ^ mt_mix(s[0], s[1]);
    }
    __syncthreads();  // every old word read before any is replaced
    const uint64_t take = std::min<uint64_t>(312, n - done);
    if (tid < 156) {
      const unsigned long long n0 = b0 ^ mt_mix(a0, a1);
      const unsigned long long n2 = n0 ^ mt_mix(b0, b1);
      s[tid] = n0;
      s[tid + 156] = n2;
      if (tid < take) o[done + tid] = mt_temper(n0);
      if (tid + 156 < take) o[done + tid + 156] = mt_temper(n2);
    }
    done += take;
    p = (uint32_t)take;
    __syncthreads();  // the new state complete before the next twist reads it
  }
  MtState* out = R.st_out + w;
  for (uint32_t i = tid; i < 312; i += blockDim.x) out->mt[i] = s[i];
  if (tid == 0) {
    out->p = p;
    out->pad = 0;
  }
}

__device__ __forceinline__ bool rejects(unsigned long long x, uint64_t n) {
  return x >= n * (0xFFFFFFFFFFFFFFFFull / n);
}

// words -> heads and tails (blockIdx.y = local worker)
__global__ void k_replay_map(ReplayDev R, SgdParams P, const uint32_t* pool,
                             const uint32_t* pool_off) {
  const uint32_t w = blockIdx.y;
  const WorkerDev W = P.workers[w];
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= W.draws) return;
  const uint32_t s = R.s;
  const unsigned long long* x = R.words + R.word_base[w] + (uint64_t)t * (1 + s);
  const uint32_t db = R.draw_base[w] + t;
  bool rej = rejects(x[0], W.n_elig);
  const uint32_t h = P.elig[W.elig_off + (uint32_t)(x[0] % W.n_elig)];
  R.heads[db] = h;
  if (P.all_but_own) {  // pool = the head's cluster (optimizer.hpp:264-277)
    const LocalCluster L = P.lclusters[P.cl_of[h]];
    for (uint32_t q = 0; q < s; ++q) {
      rej |= rejects(x[1 + q], L.count);
      R.tails[(size_t)db * s + q] = L.start + (uint32_t)(x[1 + q] % L.count);
    }
  } else {
    const uint32_t* pl = pool + pool_off[w];
    for (uint32_t q = 0; q < s; ++q) {
      rej |= rejects(x[1 + q], W.npts);
      R.tails[(size_t)db * s + q] = pl[(uint32_t)(x[1 + q] % W.npts)];
    }
  }
  if (rej) atomicOr(R.reject + w, 1u);
}

// Touch list of every draw as sort keys: slot j of draw i (0 head, then the
// neighbours in list order, then the tails; a point touched twice by one draw
// is listed once) -> key = its local point, value = i * T + j; plus the
// epoch's edge-updates per worker.
__global__ void __launch_bounds__(256) k_replay_touch(ReplayDev R, SgdParams P, uint32_t total) {
  // The block's touch rows (one draw per thread, T keys each) are formed in
  // shared memory — the list and tails copied in once, duplicates removed
  // there (no global reloads) — and written out as one contiguous run.
  extern __shared__ uint32_t sk[];  // blockDim.x * T
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t T = R.T, s = R.s, k = P.k, NONE = R.n_loc;
  // edge-updates of the epoch per worker, |N(head)| + s per draw (warp-aggregated)
  {
    uint32_t w = 0, e = 0;
    if (i < total) {
      while (w + 1 < R.nwl && R.draw_base[w + 1] <= i) ++w;
      e = (P.ncnt ? P.ncnt[R.heads[i]] : k) + s;
    }
    const uint32_t same = __match_any_sync(0xffffffffu, w);
    const uint32_t sum = __reduce_add_sync(same, e);
    if ((threadIdx.x & 31) == (uint32_t)(__ffs(same) - 1) && sum)
      atomicAdd(R.edges + w, (unsigned long long)sum);
  }
  if (i < total) {
    const uint32_t h = R.heads[i];
    uint32_t* key = sk + threadIdx.x * T;
    const uint32_t cnt = P.ncnt ? P.ncnt[h] : k;
    const uint32_t* nb = P.ell + (size_t)h * P.kpad;
    key[0] = h;
    for (uint32_t j = 1; j <= cnt; ++j) key[j] = nb[j - 1];
    for (uint32_t j = cnt + 1; j < 1 + k; ++j) key[j] = NONE;
    const uint32_t* tails = R.tails + (size_t)i * s;
    for (uint32_t q = 0; q < s; ++q) key[1 + k + q] = tails[q];
    // a point touched twice by one draw is listed at its first slot only:
    // build_knn's lists hold distinct points other than the head, a caller's
    // graph may repeat one (the reference then applies both updates in turn).
    // Comparing against already-cleared slots is harmless: the first
    // occurrence of every point is kept.
    for (uint32_t j = 1; j <= cnt; ++j) {
      const uint32_t v = key[j];
      bool dup = v == h;
      for (uint32_t a = 1; a < j && !dup; ++a) dup = key[a] == v;
      if (dup) key[j] = NONE;
    }
    for (uint32_t q = 0; q < s; ++q) {
      const uint32_t v = key[1 + k + q];
      bool dup = v == h;
      for (uint32_t a = 1; a <= cnt && !dup; ++a) dup = key[a] == v;
      for (uint32_t a = 0; a < q && !dup; ++a) dup = key[1 + k + a] == v;
      if (dup) key[1 + k + q] = NONE;
    }
  }
  __syncthreads();
  const uint32_t i0 = blockIdx.x * blockDim.x;
  if (i0 >= total) return;
  const uint32_t m = min(blockDim.x, total - i0) * T;
  const size_t base = (size_t)i0 * T;
  for (uint32_t e = threadIdx.x; e < m; e += blockDim.x) {
    R.tkey[base + e] = sk[e];
    R.tval[base + e] = (uint32_t)(base + e);  // draw * T + slot
    if (R.link) R.link[base + e] = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
    else R.pred[base + e] = 0xFFFFFFFFu;
  }
}

// After the stable sort by point: each touch's predecessor is the previous
// entry of the same point (draw order is kept inside a point's run).
__global__ void k_replay_pred(ReplayDev R, uint64_t items) {
  const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (e >= items) return;
  const uint32_t v = R.tkey[e];
  if (v == R.n_loc) return;
  uint32_t pd = 0xFFFFFFFFu;
  if (e > 0 && R.tkey[e - 1] == v)
    pd = R.tval[e - 1] / R.T - R.pt_base[v];  // the worker's draw t of the previous touch
  if (R.link) {  // one record per touch: predecessor and successor together
    const uint32_t nx = (e + 1 < items && R.tkey[e + 1] == v) ? R.tval[e + 1] : 0xFFFFFFFFu;
    if (pd != 0xFFFFFFFFu || nx != 0xFFFFFFFFu) R.link[R.tval[e]] = make_uint2(pd, nx);
  } else if (pd != 0xFFFFFFFFu) {
    R.pred[R.tval[e]] = pd;
  }
}

// ------------------------------------------------------ dataflow SGD
__device__ __forceinline__ double2 ldpos(const double2* p) { return __ldcg(p); }

__device__ __forceinline__ uint32_t ld_acquire_u8(const uint8_t* p) {
  uint16_t v;
  asm volatile("ld.acquire.gpu.global.u8 %0, [%1];" : "=h"(v) : "l"(p) : "memory");
  return v & 0xFF;
}
__device__ __forceinline__ void st_release_u8(uint8_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u8 [%0], %1;" ::"l"(p), "h"((uint16_t)v) : "memory");
}
// Position mailboxes of the warp form: the draw that last touched a point
// stores its new position straight into the slot of the point's next touch;
// each 8-byte half is single-copy atomic and starts as all-ones (a NaN no
// arithmetic produces), so a half is final once it differs from that.
constexpr unsigned long long kMboxEmpty = ~0ull;
__device__ __forceinline__ bool mbox_take(const double2* mb, double2& v) {
  unsigned long long x, y;
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(mb) : "memory");
  if (x == kMboxEmpty || y == kMboxEmpty) return false;
  v = make_double2(__longlong_as_double((long long)x), __longlong_as_double((long long)y));
  return true;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const void* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(void* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void mbox_put(double2* mb, double2 v) {
  asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(mb),
               "l"((unsigned long long)__double_as_longlong(v.x)),
               "l"((unsigned long long)__double_as_longlong(v.y))
               : "memory");
}
// A forwarded position whose bits happen to be the empty pattern (only an
// all-ones NaN, e.g. one passed in unchanged by a caller's layout) is sent as
// another NaN so the reader is never left waiting.
__device__ __forceinline__ void mbox_forward(double2* mb, double2 v) {
  const long long nan = 0x7FFFFFFFFFFFFFFFll;
  if (__double_as_longlong(v.x) == (long long)kMboxEmpty) v.x = __longlong_as_double(nan);
  if (__double_as_longlong(v.y) == (long long)kMboxEmpty) v.y = __longlong_as_double(nan);
  mbox_put(mb, v);
}

__global__ void __launch_bounds__(256) k_sgd_dataflow(SgdParams P, ReplayDev R) {
  extern __shared__ __align__(16) double sm[];
  const uint32_t k = P.k, s = P.s, C = P.n_clusters, T = R.T;
  double* wt = sm;
  double* cms = sm + (k + 1) * k;  // 3*C: mu.x, mu.y, p (or the global [C][3] table)
  for (uint32_t i = threadIdx.x; i < (k + 1) * k; i += blockDim.x) wt[i] = P.wtab[i];
  if (!P.gcells)
    for (uint32_t r = threadIdx.x; r < C; r += blockDim.x) {
      cms[3 * r] = P.means[r].x;
      cms[3 * r + 1] = P.means[r].y;
      cms[3 * r + 2] = P.cell_probs[r];
    }
  const double* cm = P.gcells ? P.cm3 : cms;
  __syncthreads();
  const double M = (double)P.m_total;
  const uint32_t stride = 2 + k + s;
  // (fallback for 1 + k + s > 32) warps claim 32 consecutive draws of a
  // worker in worker-interleaved order, one per lane; claims follow draw
  // order, so a draw only waits on draws already claimed by running warps
  const uint32_t lane = threadIdx.x & 31;
  for (;;) {
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(R.ticket, 1u);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= R.total_chunks) break;
    const uint32_t w = c % R.nwl;
    const uint32_t t = (c / R.nwl) * 32 + lane;
    const WorkerDev W = P.workers[w];
    bool pending = t < W.draws;
    const uint32_t i = R.draw_base[w] + t;  // global draw index
    const uint32_t* pr = R.pred + (size_t)i * T;
    uint32_t jj = 0, spins = 0, nap = 64;
    while (__any_sync(0xffffffffu, pending)) {
      if (!pending) continue;
      bool ready = true;
      for (; jj < T; ++jj) {
        const uint32_t q = pr[jj];
        if (q != 0xFFFFFFFFu &&
            *reinterpret_cast<volatile const uint8_t*>(R.done + R.draw_base[w] + q) == 0) {
          ready = false;
          break;
        }
      }
      if (!ready) {
        // watchdog: a predecessor is always an earlier draw of a running
        // warp, so this only fires on a schedule bug; report, never hang
        if (*reinterpret_cast<volatile uint32_t*>(R.stall) || ++spins > (1u << 22)) {
          atomicExch(R.stall, 1u);
          pending = false;
          continue;
        }
        __nanosleep(nap);  // exponential backoff (see the warp form)
        nap = min(nap * 2, 2048u);
        continue;
      }
      nap = 64;
      __threadfence();  // the predecessors' position writes before our reads
      const uint32_t head = R.heads[i];
      const uint32_t* tails = R.tails + (size_t)i * s;
      const uint32_t cnt = P.ncnt ? P.ncnt[head] : k;
      const uint32_t* nb = P.ell + (size_t)head * P.kpad;
      // every slot's position (head, neighbours, tails), loads in flight together
      uint32_t sid[1 + 64 + 16];
      double2 sp[1 + 64 + 16];
      const uint32_t nsl = 1 + cnt + s;
      for (uint32_t u = 0; u < nsl; ++u)
        sid[u] = u == 0 ? head : (u <= cnt ? nb[u - 1] : tails[u - 1 - cnt]);
      for (uint32_t u = 0; u < nsl; ++u) sp[u] = ldpos(P.pos + sid[u]);
      const double2 h = sp[0];
      // noise terms (objective.hpp:113-145)
      uint32_t own = 0;
      double lm = W.local_mass;
      if (P.all_but_own) {
        own = P.lclusters[P.cl_of[head]].gid;
        lm = P.cell_probs[own];
      }
      double remote_sum = 0.0;
      const uint32_t nr = P.all_but_own ? C : W.n_rem;
      for (uint32_t q = 0; q < nr; ++q) {
        const uint32_t r = P.all_but_own ? q : P.remote_ids[W.rem_off + q];
        if (P.all_but_own && r == own) continue;
        const double qr = cauchy_rn(h.x, h.y, cm[3 * r], cm[3 * r + 1]);
        remote_sum = __dadd_rn(remote_sum, __dmul_rn(cm[3 * r + 2], qr));
      }
      const double mean_field = __dmul_rn(M, remote_sum);
      const double sf = __ddiv_rn(__dmul_rn(M, lm), (double)s);
      double qsum = 0.0;
      for (uint32_t q = 0; q < s; ++q) {
        const double2 o = sp[1 + cnt + q];
        qsum = __dadd_rn(qsum, cauchy_rn(h.x, h.y, o.x, o.y));
      }
      const double bg = __dadd_rn(mean_field, __dmul_rn(sf, qsum));
      // attraction (objective.hpp:197-213)
      const double* wrow = wt + cnt * k;
      double loss = 0.0, bgs = 0.0, gx = 0.0, gy = 0.0;
      double gn[2 * 64];
      for (uint32_t j = 0; j < cnt; ++j) {
        const double2 o = sp[1 + j];
        const double q = cauchy_rn(h.x, h.y, o.x, o.y);
        const double wj = wrow[j];
        const double qb = __dadd_rn(q, bg);
        loss = __dadd_rn(loss, __dmul_rn(wj, -log(__ddiv_rn(q, qb))));
        bgs = __dadd_rn(bgs, __ddiv_rn(wj, qb));
        const double pull = __dmul_rn(
            __dmul_rn(__dmul_rn(__dmul_rn(2.0, wj),
                                __dsub_rn(__ddiv_rn(1.0, q), __ddiv_rn(1.0, qb))),
                      q),
            q);
        const double dx = __dsub_rn(h.x, o.x), dy = __dsub_rn(h.y, o.y);
        gx = __dadd_rn(gx, __dmul_rn(pull, dx));
        gy = __dadd_rn(gy, __dmul_rn(pull, dy));
        gn[2 * j] = __dmul_rn(-pull, dx);
        gn[2 * j + 1] = __dmul_rn(-pull, dy);
      }
      // negative repulsion (objective.hpp:216-226)
      double gm[2 * 16];
      for (uint32_t q = 0; q < s; ++q) {
        const double2 o = sp[1 + cnt + q];
        const double qn = cauchy_rn(h.x, h.y, o.x, o.y);
        const double push = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, bgs), sf), qn), qn);
        const double dx = __dsub_rn(h.x, o.x), dy = __dsub_rn(h.y, o.y);
        gx = __dsub_rn(gx, __dmul_rn(push, dx));
        gy = __dsub_rn(gy, __dmul_rn(push, dy));
        gm[2 * q] = __dmul_rn(push, dx);
        gm[2 * q + 1] = __dmul_rn(push, dy);
      }
      // mean repulsion (objective.hpp:229-236)
      for (uint32_t q = 0; q < nr; ++q) {
        const uint32_t r = P.all_but_own ? q : P.remote_ids[W.rem_off + q];
        if (P.all_but_own && r == own) continue;
        const double mx = cm[3 * r], my = cm[3 * r + 1];
        const double qr = cauchy_rn(h.x, h.y, mx, my);
        const double push = __dmul_rn(
            __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, bgs), M), cm[3 * r + 2]), qr), qr);
        gx = __dsub_rn(gx, __dmul_rn(push, __dsub_rn(h.x, mx)));
        gy = __dsub_rn(gy, __dmul_rn(push, __dsub_rn(h.y, my)));
      }
      P.loss_slot[i] = loss;
      // apply (optimizer.hpp:215-227, :293-303): head, neighbours, tails
      // updates in slot order on the preloaded positions; a point in several
      // slots continues from its first slot's running value, and every
      // distinct point is stored once at the end
      const double st = P.step;
      const uint32_t na = P.head_only ? 1 : nsl;
      for (uint32_t u = 0; u < na; ++u) {
        const double ax = u == 0 ? gx : (u <= cnt ? gn[2 * (u - 1)] : gm[2 * (u - 1 - cnt)]);
        const double ay = u == 0 ? gy : (u <= cnt ? gn[2 * (u - 1) + 1] : gm[2 * (u - 1 - cnt) + 1]);
        uint32_t f = 0;
        while (sid[f] != sid[u]) ++f;
        double2 v = sp[f];
        v.x = __dsub_rn(v.x, __dmul_rn(st, ax));
        v.y = __dsub_rn(v.y, __dmul_rn(st, ay));
        sp[f] = v;
        if (diverged(v.x, v.y))
          atomicMin(P.diverge + w, ((unsigned long long)t * stride + u) << 32 | sid[u]);
      }
      for (uint32_t u = 0; u < na; ++u) {
        uint32_t f = 0;
        while (sid[f] != sid[u]) ++f;
        if (f == u) __stcg(P.pos + sid[u], sp[u]);
      }
      __threadfence();  // our writes before the flag
      *reinterpret_cast<volatile uint8_t*>(R.done + i) = 1;
      pending = false;
    }
  }
}

// Warp-per-draw form (1 + k + s <= 32: the default k = 15, s = 5): lane u
// owns update slot u (0 head, 1..cnt neighbours, then tails) and its pred
// slot; every term is computed on its lane with the reference's operations,
// staged in the warp's shared scratch, and every lane accumulates the sums in
// the reference's order from broadcast reads over warp-uniform bounds (SURVEY
// Appendix A), so all lanes hold bits identical to the sequential loop while
// one draw's ~100 divisions run 32-wide. (Chains read through shuffles cost
// a shuffle round trip per term; profiles/r2_replay_chain.txt.)
constexpr uint32_t kDfBatch = 8;  // R.total_chunks granularity reported for the warp form

// Chains of the warp form: acc[c] = acc[c] (+|-) v[c][j] for j in [j0, j1)
// in ascending j — the reference's summation order. Terms sit in the warp's
// shared scratch (broadcast reads), 32 entries per array followed by 8
// entries that stay zero; terms the reference skips are staged as +0.0.
// Batches of 8 issue their loads together (one shared-memory latency covers
// 8 dependent adds) and run unpredicated past j1 into zeros: adding or
// subtracting +0.0 leaves every value unchanged except an accumulator of
// -0.0 under addition, and an accumulator that starts at +0.0 never becomes
// -0.0 (in round-to-nearest a sum is -0.0 only if both operands are), so the
// padded chains give the reference's bits.
constexpr uint32_t kDfScr = 40;  // doubles per scratch array
template <int NC, bool SUB>
__device__ __forceinline__ void df_chains(double (&acc)[NC], const double* const (&v)[NC],
                                          uint32_t j0, uint32_t j1) {
  for (uint32_t j = j0; j < j1; j += 8) {
    double x[NC][8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int c = 0; c < NC; ++c) x[c][e] = v[c][j + e];
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int c = 0; c < NC; ++c)
        acc[c] = SUB ? __dsub_rn(acc[c], x[c][e]) : __dadd_rn(acc[c], x[c][e]);
  }
}

#ifndef DF_MINB
#define DF_MINB 3  // min resident blocks per SM of the warp form (register cap: 80)
#endif
__global__ void __launch_bounds__(256, DF_MINB) k_sgd_dataflow_warp(SgdParams P, ReplayDev R) {
  extern __shared__ __align__(16) double sm[];
  const uint32_t k = P.k, s = P.s, C = P.n_clusters, T = R.T;
  double* wt = sm;
  double* cms = sm + (k + 1) * k;
  const size_t tab = (size_t)(k + 1) * k + (P.gcells ? 0 : 3 * (size_t)C);
  double* scr = sm + ((tab + 1) & ~(size_t)1) + (threadIdx.x >> 5) * 4 * kDfScr;
  double *sa = scr, *sb = scr + kDfScr, *sc = scr + 2 * kDfScr, *sd = scr + 3 * kDfScr;
  if ((threadIdx.x & 31) < 8)  // the zero tails of the four arrays (never written again)
    for (int a = 0; a < 4; ++a) scr[a * kDfScr + 32 + (threadIdx.x & 31)] = 0.0;
  for (uint32_t i = threadIdx.x; i < (k + 1) * k; i += blockDim.x) wt[i] = P.wtab[i];
  if (!P.gcells)
    for (uint32_t r = threadIdx.x; r < C; r += blockDim.x) {
      cms[3 * r] = P.means[r].x;
      cms[3 * r + 1] = P.means[r].y;
      cms[3 * r + 2] = P.cell_probs[r];
    }
  const double* cm = P.gcells ? P.cm3 : cms;
  __syncthreads();
  constexpr uint32_t FULL = 0xffffffffu;
  const double M = (double)P.m_total;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t stride = 2 + k + s;
  const double st = P.step;
  // Static round-robin: warp g runs the worker-interleaved draw sequence
  // g, g + nwarps, ... in order. Every draw's predecessors are earlier
  // draws, so the smallest unfinished draw is always runnable on its
  // (resident: cooperative launch) warp — no claim counter, and a waiting
  // draw holds up only its own warp.
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gw < R.followers) {
    // Loss follower: worker w's per-draw losses summed in draw order
    // (optimizer.hpp:289-290) as the draws complete, 32 slots at a time; a
    // slot holds all-ones bits until its draw writes it, and is emptied again
    // here for the next epoch. Off every dependency chain: draws never wait
    // for a follower.
    for (uint32_t w = gw; w < R.nwl; w += R.followers) {
      const uint32_t D = P.workers[w].draws;
      double* ls = P.loss_slot + R.draw_base[w];
      double acc = 0.0;
      for (uint32_t t0 = 0; t0 < D; t0 += 32) {
        const uint32_t t = t0 + lane;
        double v = 0.0;
        bool ok = t >= D;
        uint32_t spins = 0, nap = min(64u, R.nap_cap);
        for (;;) {
          if (!ok) {
            const unsigned long long b = ld_relaxed_u64(ls + t);
            if (b != kMboxEmpty) {
              v = __longlong_as_double((long long)b);
              ok = true;
            }
          }
          if (__all_sync(FULL, ok)) break;
          if ((++spins & 63) == 0 &&
              (*reinterpret_cast<volatile uint32_t*>(R.stall) || spins > (1u << 24)))
            break;  // a stalled epoch: the trainer reports it
          __nanosleep(nap);
          nap = min(nap * 2, R.nap_cap);
        }
        if (t < D) st_relaxed_u64(ls + t, kMboxEmpty);
        sa[lane] = v;
        __syncwarp();
        double a[1] = {acc};
        const double* const vv[1] = {sa};
        df_chains<1, false>(a, vv, 0, 32);
        acc = a[0];
        __syncwarp();
      }
      if (lane == 0) R.wloss[w] = acc;
    }
    return;
  }
  const uint64_t total = (uint64_t)R.nwl * R.max_draws;
  for (uint64_t c = gw - R.followers; c < total; c += nwarps - R.followers) {
    const uint32_t w = (uint32_t)(c % R.nwl);
    const WorkerDev W = P.workers[w];
    const uint32_t t = (uint32_t)(c / R.nwl);
    if (t >= W.draws) continue;
    const uint32_t i = R.draw_base[w] + t;
    // ---- everything that does not depend on positions, before any wait:
    // slot points (head, neighbours, tails), predecessor slots, weights, sf
    const uint32_t head = R.heads[i];
    const uint32_t cnt = P.ncnt ? P.ncnt[head] : k;
    const uint32_t nsl = 1 + cnt + s;
    const bool is_nb = lane >= 1 && lane <= cnt;
    const bool is_tail = lane > cnt && lane < nsl;
    uint32_t pt = head;
    if (is_nb) pt = P.ell[(size_t)head * P.kpad + lane - 1];
    else if (is_tail) pt = R.tails[(size_t)i * s + (lane - 1 - cnt)];
    // predecessor-layout lane j (touch slot j): has an earlier touch this
    // epoch (its position arrives in mailbox i*T + j), and the touch to
    // forward the new position to (none: the epoch's last touch -> pos)
    const uint2 lk = lane < T ? R.link[(size_t)i * T + lane] : make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
    const bool has_pred = lk.x != 0xFFFFFFFFu;
    const uint32_t succ = lk.y;
    double2* const myb = R.mbox + ((size_t)i * T + lane);  // this lane's mailbox
    uint32_t own = 0;
    double lm = W.local_mass;
    if (P.all_but_own) {
      own = P.lclusters[P.cl_of[head]].gid;
      lm = P.cell_probs[own];
    }
    const uint32_t nr = P.all_but_own ? C : W.n_rem;
    const double sf = __ddiv_rn(__dmul_rn(M, lm), (double)s);
    const double wj = is_nb ? wt[cnt * k + lane - 1] : 0.0;
#ifdef DF_TRACE  // per-stage SM cycles of sampled draws (diagnostic build only)
    long long tr[8];
    tr[0] = clock64();
#define DF_MARK(j) tr[j] = clock64()
#else
#define DF_MARK(j)
#endif
    // Wait until the positions of the predecessor lanes in `mine` have been
    // forwarded into their mailboxes (the values themselves: no flag, no
    // fence). Returns true when the watchdog fired (a schedule bug: report,
    // never hang).
    double2 got = make_double2(0.0, 0.0);
    auto wait_for = [&](bool mine) -> bool {
      uint32_t spins = 0, nap = min(64u, R.nap_cap);
      bool abort = false, ok = !mine || !has_pred;
      for (;;) {
        if (!ok) ok = mbox_take(myb, got);
        if (__all_sync(FULL, ok)) break;
        if ((++spins & 63) == 0 &&
            (*reinterpret_cast<volatile uint32_t*>(R.stall) || spins > (1u << 22))) {
          abort = true;
          break;
        }
        // exponential back-off: thousands of waiting warps share L2
        __nanosleep(nap);
        nap = min(nap * 2, R.nap_cap);
      }
      if (__any_sync(FULL, abort)) {
        if (lane == 0) atomicExch(R.stall, 1u);
        return true;
      }
      return false;
    };
    // ---- phase A: the head and the tails. Everything up to bg depends only
    // on them (and the epoch's cell means), so it overlaps the wait for the
    // neighbours — in the kNN graph the long dependency chains run through
    // heavily listed points, i.e. through neighbour slots. Slot lanes: 0 head,
    // 1..cnt neighbours, cnt+1.. tails; predecessor lanes follow the touch
    // layout of k_replay_touch (0 head, 1..k neighbour slots, 1+k.. tails)
    // and a repeated point carries its predecessor on its first slot only, so
    // a neighbour slot holding a tail's point belongs to phase A as well.
    const uint32_t tailmask = __ballot_sync(FULL, is_tail);
    const uint32_t grp = __match_any_sync(FULL, lane < nsl ? pt : 0xFFFFFFFFu);
    const bool needA = lane < nsl && (lane == 0 || (grp & (tailmask | 1u)) != 0);
    uint32_t sl = lane;  // predecessor lane -> slot lane
    if (lane > k && lane < 1 + k + s) sl = 1 + cnt + (lane - 1 - k);
    else if (lane > cnt && lane <= k) sl = 0;  // padded neighbour slots (no predecessor)
    const bool predA = __shfl_sync(FULL, needA, sl & 31);
    // slot lane -> its predecessor-layout lane; the first slot lane of each
    // point's group holds the point's touch (the repeats carry none)
    const uint32_t pl = lane == 0 ? 0u : (lane <= cnt ? lane : 1 + k + (lane - 1 - cnt));
    const uint32_t fl = (uint32_t)(__ffs(grp) - 1);
    const uint32_t fwd = __shfl_sync(FULL, succ, pl & 31);  // for the group's first lane
    // apply grouping (positions not needed): a point in several slots gets
    // its updates in slot order from the lane of its first slot
    const bool slot = lane < nsl && (lane == 0 || !P.head_only);
    const uint32_t act = __ballot_sync(FULL, slot);
    const uint32_t same = __match_any_sync(FULL, slot ? pt : 0xFFFFFFFFu) & act;
    // a slot's position: forwarded by the predecessor touch, or (the epoch's
    // first touch of the point) the position array; repeats copy their first
    auto position = [&](bool phase, double2& pv) {
      const double fx = __shfl_sync(FULL, got.x, pl & 31), fy = __shfl_sync(FULL, got.y, pl & 31);
      const bool fp = __shfl_sync(FULL, has_pred, pl & 31);
      double2 v = pv;
      if (phase && lane == fl) v = fp ? make_double2(fx, fy) : ldpos(P.pos + pt);
      const double vx = __shfl_sync(FULL, v.x, fl), vy = __shfl_sync(FULL, v.y, fl);
      if (phase) pv = make_double2(vx, vy);
    };
    if (wait_for(predA)) continue;
    double2 pv = make_double2(0.0, 0.0);
    position(needA, pv);
    const double hx = __shfl_sync(FULL, pv.x, 0), hy = __shfl_sync(FULL, pv.y, 0);
    DF_MARK(1);
    // noise terms (objective.hpp:113-145): terms on their lanes, every sum in
    // the reference's order by every lane from the staged terms
    // (the first 64 cells also keep q_r, p_r and h - mu_r for the mean
    // repulsion, which then needs only bgs after the neighbours arrive)
    double remote_sum = 0.0;
    double cq0 = 0.0, cp0 = 0.0, cdx0 = 0.0, cdy0 = 0.0, cq1 = 0.0, cp1 = 0.0, cdx1 = 0.0,
           cdy1 = 0.0;
    uint32_t cu0 = 0u, cu1 = 0u;
    for (uint32_t q0 = 0; q0 < nr; q0 += 32) {
      const uint32_t q = q0 + lane;
      double term = 0.0;
      bool use = false;
      if (q < nr) {
        const uint32_t r = P.all_but_own ? q : P.remote_ids[W.rem_off + q];
        if (!(P.all_but_own && r == own)) {
          const double mx = cm[3 * r], my = cm[3 * r + 1], pr = cm[3 * r + 2];
          const double qr = cauchy_rn(hx, hy, mx, my);
          term = __dmul_rn(pr, qr);
          use = true;
          if (q0 == 0) {
            cq0 = qr;
            cp0 = pr;
            cdx0 = __dsub_rn(hx, mx);
            cdy0 = __dsub_rn(hy, my);
          } else if (q0 == 32) {
            cq1 = qr;
            cp1 = pr;
            cdx1 = __dsub_rn(hx, mx);
            cdy1 = __dsub_rn(hy, my);
          }
        }
      }
      const uint32_t um = __ballot_sync(FULL, use);
      if (q0 == 0) cu0 = um;
      else if (q0 == 32) cu1 = um;
      sa[lane] = term;
      __syncwarp();
      double acc[1] = {remote_sum};
      const double* const v[1] = {sa};
      df_chains<1, false>(acc, v, 0, min(32u, nr - q0));  // skipped cells staged as 0
      remote_sum = acc[0];
      __syncwarp();
    }
    const double mean_field = __dmul_rn(M, remote_sum);
    const double qn = is_tail ? cauchy_rn(hx, hy, pv.x, pv.y) : 0.0;
    double qsum;
    {
      sa[lane] = qn;
      __syncwarp();
      double acc[1] = {0.0};
      const double* const v[1] = {sa};
      df_chains<1, false>(acc, v, cnt + 1, nsl);
      qsum = acc[0];
      __syncwarp();
    }
    const double bg = __dadd_rn(mean_field, __dmul_rn(sf, qsum));
    DF_MARK(2);
    // ---- phase B: the neighbours
    if (wait_for(!predA)) continue;
    position(lane < nsl && !needA, pv);
    DF_MARK(3);
    // attraction (objective.hpp:197-213), neighbour j on lane 1 + j
    // (the loss terms wj * -log(q / qb) feed no position: formed after the release)
    double ax = 0.0, ay = 0.0, q = 1.0, qb = 1.0, tb = 0.0, tx = 0.0, ty = 0.0;
    if (is_nb) {
      q = cauchy_rn(hx, hy, pv.x, pv.y);
      qb = __dadd_rn(q, bg);
      // wj / qb, 1 / qb and 1 / q: the three fast paths overlap (one branch)
      double iqb, iq, iq2;
      bool o1, o2;
      ddiv2_fp(wj, 1.0, qb, tb, iqb, o1);
      ddiv2_fp(1.0, 1.0, q, iq, iq2, o2);
      if (!(o1 && o2)) {
        tb = __ddiv_rn(wj, qb);
        iqb = __ddiv_rn(1.0, qb);
        iq = __ddiv_rn(1.0, q);
      }
      const double pull =
          __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, wj), __dsub_rn(iq, iqb)), q), q);
      const double dx = __dsub_rn(hx, pv.x), dy = __dsub_rn(hy, pv.y);
      tx = __dmul_rn(pull, dx);
      ty = __dmul_rn(pull, dy);
      ax = __dmul_rn(-pull, dx);
      ay = __dmul_rn(-pull, dy);
    }
    // A neighbour slot whose point no other slot of this draw holds is final
    // now (its update needs neither bgs nor the head's sums): forward it at
    // once — the long chains of the kNN graph run through neighbour slots.
    const bool solo = is_nb && grp == (1u << lane);
    if (solo) {
      double2 v = pv;
      if (slot) {
        v.x = __dsub_rn(v.x, __dmul_rn(st, ax));
        v.y = __dsub_rn(v.y, __dmul_rn(st, ay));
        if (diverged(v.x, v.y))
          atomicMin(P.diverge + w, ((unsigned long long)t * stride + lane) << 32 | pt);
      }
      if (fwd != 0xFFFFFFFFu) mbox_forward(R.mbox + fwd, v);
      else __stcg(P.pos + pt, v);
    }
    double bgs, gx, gy;
    {
      sb[lane] = tb;
      sc[lane] = tx;
      sd[lane] = ty;
      __syncwarp();
      double acc[3] = {0.0, 0.0, 0.0};  // three independent chains, list order
      const double* const v[3] = {sb, sc, sd};
      df_chains<3, false>(acc, v, 1, cnt + 1);
      bgs = acc[0];
      gx = acc[1];
      gy = acc[2];
      __syncwarp();
    }
    DF_MARK(4);
    // negative repulsion (objective.hpp:216-226), tail q on lane 1 + cnt + q
    if (is_tail) {
      const double push = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, bgs), sf), qn), qn);
      const double dx = __dsub_rn(hx, pv.x), dy = __dsub_rn(hy, pv.y);
      ax = __dmul_rn(push, dx);
      ay = __dmul_rn(push, dy);
    }
    {
      sa[lane] = ax;  // tails' pushes, subtracted in draw order
      sb[lane] = ay;
      __syncwarp();
      double acc[2] = {gx, gy};
      const double* const v[2] = {sa, sb};
      df_chains<2, true>(acc, v, cnt + 1, nsl);
      gx = acc[0];
      gy = acc[1];
      __syncwarp();
    }
    // mean repulsion (objective.hpp:229-236), q_r recomputed per cell
    const double bgsM = __dmul_rn(__dmul_rn(2.0, bgs), M);
    for (uint32_t q0 = 0; q0 < nr; q0 += 32) {
      const uint32_t q = q0 + lane;
      double px = 0.0, py = 0.0;
      uint32_t um;
      if (q0 < 64) {  // factors from phase A
        const bool b = q0 != 0;
        um = b ? cu1 : cu0;
        if ((um >> lane) & 1u) {
          const double qr = b ? cq1 : cq0;
          const double push = __dmul_rn(__dmul_rn(__dmul_rn(bgsM, b ? cp1 : cp0), qr), qr);
          px = __dmul_rn(push, b ? cdx1 : cdx0);
          py = __dmul_rn(push, b ? cdy1 : cdy0);
        }
      } else {
        bool use = false;
        if (q < nr) {
          const uint32_t r = P.all_but_own ? q : P.remote_ids[W.rem_off + q];
          if (!(P.all_but_own && r == own)) {
            const double mx = cm[3 * r], my = cm[3 * r + 1];
            const double qr = cauchy_rn(hx, hy, mx, my);
            const double push = __dmul_rn(__dmul_rn(__dmul_rn(bgsM, cm[3 * r + 2]), qr), qr);
            px = __dmul_rn(push, __dsub_rn(hx, mx));
            py = __dmul_rn(push, __dsub_rn(hy, my));
            use = true;
          }
        }
        um = __ballot_sync(FULL, use);
      }
      sa[lane] = px;
      sb[lane] = py;
      __syncwarp();
      double acc[2] = {gx, gy};
      const double* const v[2] = {sa, sb};
      df_chains<2, true>(acc, v, 0, min(32u, nr - q0));
      gx = acc[0];
      gy = acc[1];
      __syncwarp();
    }
    DF_MARK(5);
    if (lane == 0) {
      ax = gx;
      ay = gy;
    }
    // ---- apply (optimizer.hpp:215-227, :293-303): head, neighbours, tails;
    // the first lane of each point's group applies its slots' updates in slot
    // order and forwards the result to the point's next touch (or stores it)
    sa[lane] = ax;
    sb[lane] = ay;
    __syncwarp();
    DF_MARK(6);
    if (lane < nsl && lane == fl && !solo) {
      double2 v = pv;
      if (slot)
        for (uint32_t m = same; m; m &= m - 1) {
          const uint32_t u = __ffs(m) - 1;
          v.x = __dsub_rn(v.x, __dmul_rn(st, sa[u]));
          v.y = __dsub_rn(v.y, __dmul_rn(st, sb[u]));
          if (diverged(v.x, v.y))
            atomicMin(P.diverge + w, ((unsigned long long)t * stride + u) << 32 | pt);
        }
      if (fwd != 0xFFFFFFFFu) mbox_forward(R.mbox + fwd, v);
      else __stcg(P.pos + pt, v);
    }
    // every mailbox is read once: empty it again for the next epoch (no
    // per-epoch fill), off the dependency chain
    if (has_pred)
      mbox_put(myb, make_double2(__longlong_as_double((long long)kMboxEmpty),
                                       __longlong_as_double((long long)kMboxEmpty)));
    __syncwarp();  // the updates read from the scratch before it is reused
    // the draw's loss (objective.hpp:197-213): sum over the list in order
    {
      sa[lane] = is_nb ? __dmul_rn(wj, -log(__ddiv_rn(q, qb))) : 0.0;
      __syncwarp();
      double acc[1] = {0.0};
      const double* const v[1] = {sa};
      df_chains<1, false>(acc, v, 1, cnt + 1);
      if (lane == 0)  // (never the all-ones pattern the loss followers wait on)
        P.loss_slot[i] = __double_as_longlong(acc[0]) == (long long)kMboxEmpty
                             ? __longlong_as_double(0x7FFFFFFFFFFFFFFFll)
                             : acc[0];
      __syncwarp();
    }
#ifdef DF_TRACE
    DF_MARK(7);
    if (lane == 0 && w == 0 && t % 2048 == 777)
      printf("dftrace t=%u waitA %lld noise %lld waitB+load %lld attract %lld repulse %lld tail %lld apply+loss %lld\n",
             t, tr[1] - tr[0], tr[2] - tr[1], tr[3] - tr[2], tr[4] - tr[3], tr[5] - tr[4],
             tr[6] - tr[5], tr[7] - tr[6]);

#endif
  }
}

// ------------------------------------------------------ host launchers
static unsigned blocks_for(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

void launch_mt_words(const ReplayDev& R, const uint64_t* counts, cudaStream_t st) {
  k_mt_words<<<R.nwl, 160, 0, st>>>(R, counts);
}

void launch_replay_map(const ReplayDev& R, const SgdParams& P, const uint32_t* pool,
                       const uint32_t* pool_off, cudaStream_t st) {
  const dim3 grid(blocks_for(std::max<uint32_t>(R.max_draws, 1), 256), R.nwl);
  k_replay_map<<<grid, 256, 0, st>>>(R, P, pool, pool_off);
}

static int bits_for(uint32_t v) {
  int b = 1;
  while (b < 32 && (v >> b)) ++b;
  return b;
}

size_t replay_sort_bytes(uint64_t items, uint32_t n_loc) {
  size_t b = 0;
  NB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                          (uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)items,
                                          0, bits_for(n_loc)));
  return b;
}

void launch_replay_deps(const ReplayDev& R, const SgdParams& P, void* sort_tmp, size_t sort_bytes,
                        cudaStream_t st) {
  const uint32_t total = R.total_draws;
  const uint64_t items = (uint64_t)total * R.T;
  if (!total) return;
  const size_t tsm = (size_t)256 * R.T * sizeof(uint32_t);
  if (tsm > 48 * 1024)
    NB_CUDA(cudaFuncSetAttribute(k_replay_touch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)tsm));
  k_replay_touch<<<blocks_for(total, 256), 256, tsm, st>>>(R, P, total);
  // stable LSD radix sort by point over the draw-ordered touches
  size_t b = sort_bytes;
  NB_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp, b, R.tkey, R.tkey2, R.tval, R.tval2,
                                          (int64_t)items, 0, bits_for(R.n_loc), st));
  ReplayDev Rs = R;
  Rs.tkey = R.tkey2;
  Rs.tval = R.tval2;
  k_replay_pred<<<blocks_for(items, 256), 256, 0, st>>>(Rs, items);
}

bool dataflow_warp_form(uint32_t k, uint32_t s) {
  static const bool thread_form = std::getenv("NOMAD_B200_DATAFLOW_THREAD") != nullptr;
  return 1 + k + s <= 32 && !thread_form;
}
uint32_t dataflow_draws_per_chunk(uint32_t k, uint32_t s) {
  return dataflow_warp_form(k, s) ? kDfBatch : 32;
}
// per-warp scratch of the warp form: 4 x kDfScr doubles (8 warps per block)
static size_t df_smem(size_t smem, uint32_t k, uint32_t s) {
  return dataflow_warp_form(k, s) ? ((smem + 15) & ~(size_t)15) + 8 * 4 * kDfScr * sizeof(double)
                                   : smem;
}

void launch_sgd_dataflow(const SgdParams& P, const ReplayDev& R, uint32_t nblocks, size_t smem,
                         cudaStream_t st) {
  const bool wf = dataflow_warp_form(P.k, P.s);
  const size_t sm = df_smem(smem, P.k, P.s);
  auto kern = wf ? k_sgd_dataflow_warp : k_sgd_dataflow;
  if (sm > 48 * 1024)
    NB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  // every block resident at once (the static schedule relies on it)
  SgdParams Pc = P;
  ReplayDev Rc = R;
  void* args[] = {&Pc, &Rc};
  NB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(nblocks), dim3(256), args, sm, st));
}

uint32_t dataflow_resident_blocks(size_t smem, int sm_count, uint32_t k, uint32_t s) {
  const bool wf = dataflow_warp_form(k, s);
  const size_t sm = df_smem(smem, k, s);
  auto kern = wf ? k_sgd_dataflow_warp : k_sgd_dataflow;
  if (sm > 48 * 1024)
    NB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per_sm = 0;
  NB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, sm));
  return (uint32_t)std::max(per_sm, 1) * (uint32_t)sm_count;
}

}  // namespace nb
