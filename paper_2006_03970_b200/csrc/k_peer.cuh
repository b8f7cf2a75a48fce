// k_peer.cuh — §8(f3) column-sharded solves with device-resident exchanges over peer memory
// ("per Newton step one exchange … a few µs with NVLS multimem or symmetric memory").
//
// Every rank (one process per GPU) allocates one exchange REGION and maps every other rank's region
// through CUDA IPC (NVLink peer memory).  A rank deposits its contribution straight into slot
// [rank] of EVERY rank's region with plain stores (P2P over NVLink), then raises its flag in every
// region; a rank that needs the sum waits until every flag of its own region has reached the
// exchange's epoch and adds the slots in rank order 0, 1, …, G−1 — so all ranks hold
// bitwise-identical sums and take identical control decisions, with no host round trip.  The
// exchanges are kernels, so they sit inside the conditional-node graph of a solve (k_ctl.cuh).
//
// Region layout (doubles unless noted):
//   flags   uint64 [kPeerMaxRanks]         flag[q] = last epoch rank q deposited (256 B)
//   cnt     int64  [kPeerMaxRanks]         gathered-column counts r_q (SMW all-gather)
//   small   [2][G][ss]                     per-evaluation records, double-buffered by epoch parity
//   big     [G][sb]                        gathered active columns (r < m) / partial Grams (r ≥ m)
// Epochs: every exchange increments the rank's device counter; all ranks run the same sequence of
// exchanges (their control decisions are identical), so epoch e names the same exchange everywhere.
// A rank cannot complete exchange e + 1 before every rank deposited e + 1, which each rank does
// only after it has consumed exchange e (stream order).  Hence a rank is at most one exchange
// ahead of any other: flags are compared with ≥, consecutive small exchanges (Armijo backtracks)
// alternate parities, and the big slots — always separated by at least one small exchange
// (the trial evaluation between two Newton steps) — need a single buffer.
// Waits poll with sys-scope acquire loads and give up after kPeerTimeoutNs (error flag set: the
// solve returns SSNAL_ECUDA instead of hanging the GPU).
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"
#include "k_newton.cuh"

namespace ssn {

constexpr int kPeerMaxRanks = 16;
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000ull * 1000ull * 1000ull;  // 20 s

struct PeerComm {  // kernel parameter (by value)
  char* base[kPeerMaxRanks];  // region of every rank (this rank's own at [rank])
  int rank, size;
  int64_t ss, sb;             // doubles per small / big slot
  int64_t ccap;               // big slot capacity in columns of m doubles (gathered A_J)
  unsigned long long* epoch;  // this rank's exchange counter (device)
  unsigned* ticket;           // last-CTA counter of the multi-CTA deposits (device)
  int* err;                   // 1: a wait timed out; 2: gathered counts disagree with the global r
};

SSN_HD int64_t peer_small_off() { return 2 * kPeerMaxRanks * 8; }  // bytes: flags + cnt
SSN_HD int64_t peer_big_off(int size, int64_t ss) { return peer_small_off() + (int64_t)2 * size * ss * 8; }
SSN_HD int64_t peer_region_bytes(int size, int64_t ss, int64_t sb) { return peer_big_off(size, ss) + (int64_t)size * sb * 8; }

SSN_DEV unsigned long long* peer_flags(const PeerComm& pc, int q) { return (unsigned long long*)pc.base[q]; }
SSN_DEV int64_t* peer_cnt(const PeerComm& pc, int q) { return (int64_t*)(pc.base[q] + kPeerMaxRanks * 8); }
// slot of rank `src` for parity p in the region of rank q
SSN_DEV double* peer_small(const PeerComm& pc, int q, int p, int src) {
  return (double*)(pc.base[q] + peer_small_off()) + ((int64_t)p * pc.size + src) * pc.ss;
}
SSN_DEV double* peer_big(const PeerComm& pc, int q, int src) {
  return (double*)(pc.base[q] + peer_big_off(pc.size, pc.ss)) + (int64_t)src * pc.sb;
}

SSN_DEV void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
SSN_DEV unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Raise this rank's flag to epoch e in every region (one thread, after its CTA's deposits were
// made visible with __threadfence_system()).
SSN_DEV void peer_signal(const PeerComm& pc, unsigned long long e) {
  __threadfence_system();
  for (int q = 0; q < pc.size; ++q) st_release_sys(peer_flags(pc, q) + pc.rank, e);
}
// Wait until every rank's flag in this rank's region is ≥ e (one thread).  false on timeout.
SSN_DEV bool peer_wait(const PeerComm& pc, unsigned long long e) {
  const unsigned long long* f = peer_flags(pc, pc.rank);
  const unsigned long long t0 = global_ns();
  for (int q = 0; q < pc.size; ++q) {
    while (ld_acquire_sys(f + q) < e) {
      if (global_ns() - t0 > kPeerTimeoutNs) {
        atomicExch(pc.err, 1);
        return false;
      }
    }
  }
  return true;
}

// ---- the evaluation record of a sharded ψ evaluation ----
// rec[k], k < m: Σ_b part_vec[b][k] over the valid rows; m ≤ k < m + 4: Σ_q part_scal[q][k − m];
// k = m + 4: the local r.  One 16-CTA cluster: CTA c takes the 32-element blocks kb ≡ c (mod 16);
// lane = element, warp w sums rows b ≡ w (mod 8) ascending (8 loads in flight), the 8 warp sums are
// added in warp order — a fixed order, so every caller that uses rec_block gets identical bits.
constexpr int kRecCS = 16;
SSN_DEV void rec_block(int kb, int64_t m, const double* __restrict__ part_vec, const int* __restrict__ valid,
                       int nparts, const double* __restrict__ part_scal, int nscal, const int64_t* __restrict__ r_dev,
                       double (*red)[32], double* out_blk) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t k = (int64_t)kb * 32 + lane;
  double s = 0.0;
  if (k < m) {
    for (int b0 = warp; b0 < nparts; b0 += 64) {
      double v[8];
      bool ok[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = b0 + 8 * u;
        ok[u] = b < nparts && (!valid || valid[b]);
        v[u] = ok[u] ? __ldcg(part_vec + (size_t)b * m + k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (ok[u]) s += v[u];
    }
  } else if (k < m + 4) {
    for (int q = warp; q < nscal; q += 8) s += part_scal[q * 4 + (k - m)];
  } else if (k == m + 4 && warp == 0) {
    s = r_dev ? (double)*r_dev : 0.0;
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    double t = red[0][lane];
    for (int w = 1; w < 8; ++w) t += red[w][lane];
    out_blk[lane] = t;
  }
  __syncthreads();
}

// Callback provider (host-driven sharded mode): the record into out (m + 5 doubles) for the
// caller's all-reduce.
__global__ void __cluster_dims__(kRecCS, 1, 1) __launch_bounds__(256)
    k_prereduce16(int64_t m, const double* __restrict__ part_vec, const int* __restrict__ valid, int nparts,
                  const double* __restrict__ part_scal, int nscal, const int64_t* __restrict__ r_dev,
                  double* __restrict__ out) {
  __shared__ double red[8][32];
  __shared__ double blk[32];
  const int nkb = (int)((m + 5 + 31) / 32);
  for (int kb = blockIdx.x; kb < nkb; kb += kRecCS) {
    rec_block(kb, m, part_vec, valid, nparts, part_scal, nscal, r_dev, red, blk);
    const int64_t k = (int64_t)kb * 32 + threadIdx.x;
    if (threadIdx.x < 32 && k < m + 5) out[k] = blk[threadIdx.x];
  }
}

// Peer provider: each CTA deposits its blocks of the record straight into slot [rank] of every
// rank's region (parity of the exchange's epoch); after a cluster barrier CTA 0 raises the flags
// and waits for every rank's; after a second barrier each CTA sums its blocks over the ranks in
// rank order into out, and the global r into rg_out.  pred (nullable): graph-mode predicate,
// uniform over the ranks (a global control decision).
__global__ void __cluster_dims__(kRecCS, 1, 1) __launch_bounds__(256)
    k_peer_eval(PeerComm pc, int64_t m, const double* __restrict__ part_vec, const int* __restrict__ valid,
                int nparts, const double* __restrict__ part_scal, int nscal, const int64_t* __restrict__ r_dev,
                double* __restrict__ out, int64_t* rg_out, const int* pred) {
  __shared__ double red[8][32];
  __shared__ double blk[32];
  if (pred && *pred == 0) return;  // uniform over the grid
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  // every CTA reads the epoch before CTA 0 advances it (the first cluster barrier orders them)
  const unsigned long long e = *(volatile unsigned long long*)pc.epoch + 1;
  const int p = (int)(e & 1);
  const int nkb = (int)((m + 5 + 31) / 32);
  for (int kb = blockIdx.x; kb < nkb; kb += kRecCS) {
    rec_block(kb, m, part_vec, valid, nparts, part_scal, nscal, r_dev, red, blk);
    const int64_t k = (int64_t)kb * 32 + threadIdx.x;
    if (threadIdx.x < 32 && k < m + 5)
      for (int q = 0; q < pc.size; ++q) peer_small(pc, q, p, pc.rank)[k] = blk[threadIdx.x];
  }
  __threadfence_system();
  cluster.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *pc.epoch = e;
    peer_signal(pc, e);
    peer_wait(pc, e);
  }
  cluster.sync();
  for (int kb = blockIdx.x; kb < nkb; kb += kRecCS) {
    const int64_t k = (int64_t)kb * 32 + threadIdx.x;
    if (threadIdx.x < 32 && k < m + 5) {
      double s = peer_small(pc, pc.rank, p, 0)[k];
      for (int q = 1; q < pc.size; ++q) s += peer_small(pc, pc.rank, p, q)[k];
      out[k] = s;
      if (k == m + 4) *rg_out = (int64_t)s;
    }
  }
}

// ---- small exchanges: one CTA ----
// Generic small all-reduce in place (count ≤ ss): op 0 = sum, 1 = max, rank order.
__global__ void __launch_bounds__(1024) k_peer_allreduce(PeerComm pc, double* buf, int64_t count, int op) {
  __shared__ unsigned long long s_e;
  const int tid = threadIdx.x;
  if (tid == 0) s_e = ++*pc.epoch;
  __syncthreads();
  const unsigned long long e = s_e;
  const int p = (int)(e & 1);
  for (int64_t k = tid; k < count; k += blockDim.x) {
    const double v = buf[k];
    for (int q = 0; q < pc.size; ++q) peer_small(pc, q, p, pc.rank)[k] = v;
  }
  __syncthreads();
  if (tid == 0) {
    peer_signal(pc, e);
    peer_wait(pc, e);
  }
  __syncthreads();
  for (int64_t k = tid; k < count; k += blockDim.x) {
    double s = peer_small(pc, pc.rank, p, 0)[k];
    for (int q = 1; q < pc.size; ++q) {
      const double v = peer_small(pc, pc.rank, p, q)[k];
      s = op == 0 ? s + v : fmax(s, v);
    }
    buf[k] = s;
  }
}

// ---- big exchanges: multi-CTA deposit (last CTA signals), then a waiting consumer ----
SSN_DEV void peer_last_cta_signal(const PeerComm& pc) {
  __shared__ bool last;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(pc.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    *pc.ticket = 0u;
    peer_signal(pc, ++*pc.epoch);
  }
}
// every CTA of a consumer: wait for the epoch the deposit kernel signalled (it ran before, in
// stream order, so *epoch is final)
SSN_DEV void peer_cta_wait(const PeerComm& pc) {
  if (threadIdx.x == 0) peer_wait(pc, *(volatile unsigned long long*)pc.epoch);
  __syncthreads();
}

// Generic big all-reduce (host-driven sharded mode): buf (count ≤ sb doubles) into every rank's big
// slot [rank] …
__global__ void k_peer_put_big(PeerComm pc, const double* __restrict__ buf, int64_t count) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
    const double v = buf[k];
    for (int q = 0; q < pc.size; ++q) peer_big(pc, q, pc.rank)[k] = v;
  }
  peer_last_cta_signal(pc);
}
// … then buf ← Σ (or max) over the ranks' slots in rank order.
__global__ void k_peer_reduce_big(PeerComm pc, double* __restrict__ buf, int64_t count, int op) {
  peer_cta_wait(pc);
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
    double s = peer_big(pc, pc.rank, 0)[k];
    for (int q = 1; q < pc.size; ++q) {
      const double v = peer_big(pc, pc.rank, q)[k];
      s = op == 0 ? s + v : fmax(s, v);
    }
    buf[k] = s;
  }
}

// A sharded Newton direction in graph mode (§8(f3)), predicated on the GLOBAL branch (geo), in two
// merged nodes (each serves both branches, so a step pays no predicated-off node for them):
//
// SMW branch (0 < r < m, Eq. (19)) — the all-gather of the active columns fused into the gather:
//   dir1: column a of this rank's local A_J goes straight to column a of big slot [rank] in EVERY
//         rank's region (capacity ccap ≥ m columns of m doubles), its count to cnt[rank]; the last
//         CTA signals;
//   dir2: one CTA waits for the gathered columns, then idx[0, rg) = the big-region column of each
//         gathered column in rank order (rank q's column i → q·ccap + i), so the SMW kernels read A_J
//         through AccA{big, m} and idx exactly as from a packed r × m buffer (counts that do not add
//         up to the global r set err = 2).
// m × m branch (r ≥ m, Eq. (18)) — the GEMM → all-gather fusion of the partial Grams:
//   k_gram_sk (raw mode, a node of its own): the local partial Gram A_J A_Jᵀ of this rank's active
//         columns into W (m × m, ld = m), as the host-driven sharded path forms it;
//   dir2: the partial deposited into big slot [rank] of every rank; the last CTA signals;
//   k_peer_gram_sum (below) then forms the Newton matrix on every rank.
template <class Acc>
__global__ void __launch_bounds__(256) k_peer_dir1(PeerComm pc, const Acc A, int64_t m, const int32_t* __restrict__ J,
                                                   const int64_t* __restrict__ r_dev, const DirGeo* geo) {
  const int br = geo->branch;
  const int64_t r = *r_dev;
  if (br == 1) {
    for (int64_t a = blockIdx.x; a < r; a += gridDim.x) {
      const auto col = A.col(J[a]);
      for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
        const double v = col.ld(k);
        for (int q = 0; q < pc.size; ++q) peer_big(pc, q, pc.rank)[a * m + k] = v;
      }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
      for (int q = 0; q < pc.size; ++q) peer_cnt(pc, q)[pc.rank] = r;
    peer_last_cta_signal(pc);
  }
}
__global__ void k_peer_dir2(PeerComm pc, const double* __restrict__ W, int64_t m, const DirGeo* geo,
                            int32_t* __restrict__ idx) {
  __shared__ int64_t off[kPeerMaxRanks + 1];
  const int br = geo->branch;
  if (br == 1) {
    if (blockIdx.x != 0) return;
    const int64_t rg = geo->r;
    peer_cta_wait(pc);
    if (threadIdx.x == 0) {
      off[0] = 0;
      for (int q = 0; q < pc.size; ++q) off[q + 1] = off[q] + *(volatile int64_t*)(peer_cnt(pc, pc.rank) + q);
      if (off[pc.size] != rg) atomicExch(pc.err, 2);
    }
    __syncthreads();
    for (int q = 0; q < pc.size; ++q)
      for (int64_t i = threadIdx.x; i < off[q + 1] - off[q] && off[q] + i < rg; i += blockDim.x)
        idx[off[q] + i] = (int32_t)(q * pc.ccap + i);
  } else if (br == 2) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m * m;
         e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = e % m, j = e / m;
      if (i < j) continue;
      const double v = W[e];  // the raw partial (lower part) of k_gram_sk
      for (int q = 0; q < pc.size; ++q) peer_big(pc, q, pc.rank)[e] = v;
    }
    peer_last_cta_signal(pc);
  }
}
// … and every rank forms M = I_m + κ Σ_q (rank order) with the jitter and the rhs row g, as
// k_gram_reduce(Σ, ns = 1, diag = 1, mult = κ) does on the summed buffer of the host-driven path.
__global__ void k_peer_gram_sum(PeerComm pc, int64_t m, double* __restrict__ M, const double* __restrict__ g,
                                const DirGeo* geo, double kappa, int64_t ld, double jit) {
  if (geo) {
    if (geo->branch != 2) return;
    kappa = geo->mult;
    ld = geo->ld;
    jit = geo->jit;
  }
  peer_cta_wait(pc);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m * m; e += (int64_t)gridDim.x * blockDim.x) {
    if (g && e < m) M[m + e * ld] = g[e];
    const int64_t i = e % m, j = e / m;
    if (i < j) continue;
    double s = 0.0;
    for (int q = 0; q < pc.size; ++q) s += peer_big(pc, pc.rank, q)[e];
    double v = kappa * s + (i == j ? 1.0 : 0.0);
    if (i == j && jit != 0.0) v = __fma_rn(v, jit, v);
    M[i + j * ld] = v;
  }
}

// ---- protocol test: G ranks emulated by G CTAs of ONE cooperative launch (co-resident) ----
// CTA q plays rank q with its own PeerComm (regions = G buffers of one allocation), and runs `iters`
// rounds of: a small exchange (values v(q, it, k)), then every third round a big exchange — the
// same deposit / signal / wait / rank-ordered sum code as the solve's exchanges.  Each rank checks
// every sum against the closed form Σ_q v(q, it, k) (integers, exact) and counts mismatches.
SSN_HD double peer_test_val(int q, int it, int64_t k) { return (double)((q + 1) * 1000003LL + it * 7919LL + k * 31LL); }
__global__ void __launch_bounds__(256) k_peer_emulate(PeerComm proto, char* const* bases, int iters, int64_t cnt,
                                                      unsigned long long* epochs, int* errs, int* mismatch,
                                                      double* last_small, double* last_big) {
  PeerComm pc = proto;
  pc.rank = blockIdx.x;
  pc.epoch = epochs + blockIdx.x;
  pc.err = errs + blockIdx.x;
  for (int q = 0; q < pc.size; ++q) pc.base[q] = bases[q];
  __shared__ unsigned long long s_e;
  int bad = 0;
  for (int it = 0; it < iters; ++it) {
    const bool big = it % 3 == 2;
    if (threadIdx.x == 0) s_e = ++*pc.epoch;
    __syncthreads();
    const unsigned long long e = s_e;
    const int p = (int)(e & 1);
    for (int64_t k = threadIdx.x; k < cnt; k += blockDim.x) {
      const double v = peer_test_val(pc.rank, it, k);
      for (int q = 0; q < pc.size; ++q) {
        if (big) peer_big(pc, q, pc.rank)[k] = v;
        else peer_small(pc, q, p, pc.rank)[k] = v;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      peer_signal(pc, e);
      peer_wait(pc, e);
    }
    __syncthreads();
    for (int64_t k = threadIdx.x; k < cnt; k += blockDim.x) {
      double s = big ? peer_big(pc, pc.rank, 0)[k] : peer_small(pc, pc.rank, p, 0)[k];
      double want = peer_test_val(0, it, k);
      for (int q = 1; q < pc.size; ++q) {
        s += big ? peer_big(pc, pc.rank, q)[k] : peer_small(pc, pc.rank, p, q)[k];
        want += peer_test_val(q, it, k);
      }
      bad += s != want;
      (big ? last_big : last_small)[pc.rank * cnt + k] = s;  // the last exchange of each kind remains
    }
    // consume before the next deposit (the production kernels get this from stream order)
    __syncthreads();
  }
  atomicAdd(mismatch, bad);
}

}  // namespace ssn
