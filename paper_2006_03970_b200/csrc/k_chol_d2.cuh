// K4, DSMEM-resident with split ownership (96 < N ≤ 512): the Cholesky factor of the N × N SPD
// matrix of Eq. (18) / (19), the forward substitution (right-hand side carried as row N) and the
// backward substitution, by one 16-CTA cluster whose shared memory holds the whole lower triangle.
//
// Ownership.  k_chol_dsm gives CTA j all of block column j, so owner j absorbs j·(T − j) tile
// updates on one SM and the middle owners fall behind the panel chain.  Here the tiles are split
// by role:
//   chain tiles (j, j) and (j + 1, j)  → CTA j mod NC  (the critical path: factor, W_j = L_jj⁻¹,
//                                         L_{j+1,j}; W_j never leaves the CTA for that TRSM);
//   trailing tiles (i, j), i ≥ j + 2   → CTA NC + ((i − j − 2) + 3j) mod (16 − NC), so the
//                                         trailing tiles of one column land on distinct CTAs.
// NC = kD2Chain = 5 chain CTAs: each chain CTA absorbs every earlier panel into its chain tiles
// between its own columns, so more chain CTAs give each more time for that look-ahead (4 → 5:
// 5% faster at N = 435–512; 6 leaves too few trailing CTAs at large N and needs 13 tile slots).
// Every CTA keeps its tiles in shared memory for the whole launch (≤ 12 × 8.4 KB).
//
// Schedule (per 128-thread quad; the tiles of a CTA alternate between its two quads, so a chain
// CTA's quad 0 holds the diagonal tiles and quad 1 the sub-diagonal ones).  For k = −1 … T − 2:
//   A: absorb the panels up to k into my tiles of column k + 1 (A_ij −= L_ik L_jkᵀ, DMMA), waiting;
//   B: finish my tiles of column k + 1 (diagonal: diag_factor4 → L_jj, W_j; else L_ij = A_ij W_jᵀ);
//   C: absorb into my tiles of later columns the panels ≤ k that are already published (no wait).
// Finished tiles are published with a release store of a per-tile flag in the owner's shared
// memory; consumers poll it with cluster-scope acquire loads, copy the B operand into a local double
// buffer and read the A fragments from the producer's shared memory.  The critical hand-off is
// pushed instead: the chain CTA of column j sends L_{j+1,j} into an inbox of the chain CTA of
// column j + 1 with one bulk DSMEM copy (cp.async.bulk shared::cta → shared::cluster, completion on
// the receiver's mbarrier), so the next diagonal update reads local memory only.  Every wait is on
// work of an earlier phase, so the schedule cannot deadlock (a cluster's CTAs are co-resident).
//
// Backward substitution v = L⁻ᵀz (z = row N of the factor), for j = T − 1 … 0 by the chain CTA of j:
//   v_j = u_j − P_jᵀ v_{j+1},  u_j = W_jᵀ(z_j − L_{j+2,j}ᵀ v_{j+2} − Σ_{i ≥ j+3} L_ijᵀ v_i),
//   P_j = L_{j+1,j} W_j (formed by idle warps after the factorisation),
// so only one 32-term dot product per lane sits between the arrival of v_{j+1} and the push of v_j.
// v_j is broadcast to every CTA by bulk copies; the trailing partials L_ijᵀ v_i (i ≥ j + 3) are
// formed by their owners as soon as v_i arrives and pushed into per-(j, i) slots (summed in fixed
// order: the result is deterministic).  Outputs as k_chol_cluster: out = scale·v,
// *dot_out = Σ dotv·out, yt = ybase + out, *info = 1 on a non-positive pivot.
#pragma once
#include <cooperative_groups.h>
#include "k_chol_dsm.cuh"

namespace ssn {

constexpr int kD2Slots = 12;  // max tiles per CTA over N ≤ 512 for 4 or 5 chain CTAs (13 for 6; tools/probes/d2_probe)
constexpr int kD2Chain = 5;   // chain CTAs (tools/probes/d2_probe: 4 / 5 / 6 chain CTAs, N = 435: 148.7 / 140.6 /
                              // 142.7 µs, N = 500: 182.7 / 173.6 / 178.1 µs)
constexpr int kD2Bytes = kTileD * 8;  // one tile (8448 B, a multiple of 16)
constexpr size_t kD2SmemDoubles = (size_t)kD2Slots * kTileD  // owned tiles
                                  + 4 * kTileD                 // W_j of my diagonal tiles (j ≡ CTA mod NC, ≤ 4)
                                  + 4 * kTileD                 // B operands (2 per quad); P_j in the backward
                                  + kTileD                     // inbox: L_{j,j−1} pushed by the previous chain CTA
                                  + kDiagScratch               // diag_factor4 scratch; partial staging later
                                  + kDsmCS * 32                // vin[i][·] = v_i
                                  + 4 * kDsmCS * 32            // pacc[q][i][·] = L_ijᵀ v_i (j = 4q + CTA)
                                  + 64                         // gᵀd partial, backward scratch
                                  + 24                         // mbarriers: inbox, v_i (16), partials (4)
                                  + 64;                        // ints: flags, tile list, slot table
constexpr size_t kD2Smem = kD2SmemDoubles * sizeof(double);

#ifdef D2_PROBE
__device__ unsigned long long g_d2[18][8];
#define D2STAMP(k, e) do { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_d2[k][e] = t_; } while (0)
#else
#define D2STAMP(k, e) do {} while (0)
#endif

// NC chain CTAs (the chain tiles of column j on CTA j mod NC; lc = the column's index on its chain
// CTA) and NT = 16 − NC trailing CTAs (tile (i, j), i ≥ j + 2, on NC + ((i − j − 2) + 3j) mod NT).
template <int NC> SSN_DEV int d2_owner(int i, int j) {
  return i - j <= 1 ? j % NC : NC + (i - j - 2 + 3 * j) % (kDsmCS - NC);
}
template <int NC> SSN_DEV int d2_lc(int j) { return j / NC; }
template <int NC> SSN_DEV int d2_col(int c, int q) { return c + NC * q; }
SSN_DEV int d2_cntm(int len, int res, int mod) { return len > res ? (len - res + mod - 1) / mod : 0; }  // #{x < len : x ≡ res (mod)}
// position of tile (i, j) in its owner's list (column-major order of the owner's tiles)
template <int NC> SSN_DEV int d2_slot(int i, int j, int ntr) {
  constexpr int NT = kDsmCS - NC;
  if (i - j <= 1) return 2 * d2_lc<NC>(j) + (i - j);
  const int h = (i - j - 2 + 3 * j) % NT;
  int s = 0;
  for (int jj = 0; jj < j; ++jj) s += d2_cntm(ntr - jj - 2, ((h - 3 * jj) % NT + NT) % NT, NT);
  return s + (i - j - 2) / NT;
}

SSN_DEV uint32_t d2_mapa(const void* p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
SSN_DEV void d2_remote_expect(uint32_t rbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(rbar), "r"(bytes)
               : "memory");
}
SSN_DEV void d2_push(uint32_t rdst, const void* src, uint32_t bytes, uint32_t rbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   rdst),
               "r"(smem_u32(src)), "r"(bytes), "r"(rbar)
               : "memory");
}
SSN_DEV void d2_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
SSN_DEV void d2_wait_reads() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
SSN_DEV bool d2_mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\n"
      "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
SSN_DEV void d2_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Σ_r M[r][lane] · x[r] (M row-major TLD in shared memory, x broadcast from shared memory)
SSN_DEV double d2_coldot(const double* M, const double* x, int lane) {
  double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int r = 0; r < CHT; ++r) s[r & 3] = fma(M[r * TLD + lane], x[r], s[r & 3]);
  return (s[0] + s[1]) + (s[2] + s[3]);
}

template <int NC>
SSN_DEV void chol_d2_body(const double* __restrict__ M, int N, int ld, double* __restrict__ out, double scale,
                          const double* __restrict__ dotv, double* dot_out, int* info,
                          const double* __restrict__ ybase, double* __restrict__ yt, const DirGeo* geo, int want,
                          int nmin, int nmax, const CholArgs* ca) {
  namespace cg = cooperative_groups;
  if (geo) {  // graph mode: predicated on the branch and on nmin ≤ N ≤ nmax (uniform over the cluster)
    if ((want >= 0 ? geo->branch != want : (geo->branch != 1 && geo->branch != 2)) || geo->N > nmax ||
        geo->N < nmin)
      return;
    if (ca) {
      const CholArgs& c = ca[geo->branch - 1];
      out = c.out;
      scale = c.scale;
      dotv = c.dotv;
      dot_out = c.dot_out;
      ybase = c.ybase;
      yt = c.yt;
    }
    N = geo->N;
    ld = geo->ld;
  }
  extern __shared__ __align__(16) double sm[];
  double* T = sm;                        // T + s·kTileD = my tile s (row-major, TLD)
  double* Wb = T + kD2Slots * kTileD;    // Wb + (j/4)·kTileD = W_j (row-major, TLD)
  double* Bq = Wb + 4 * kTileD;          // Bq + (2·quad + parity)·kTileD; backward: P_j
  double* inbox = Bq + 4 * kTileD;       // L_{j,j−1} (chain CTAs)
  double* dscr = inbox + kTileD;         // diag_factor4 scratch; backward: partial staging (slot·32)
  double* vin = dscr + kDiagScratch;     // vin[i·32 + r] = v_i[r]
  double* pacc = vin + kDsmCS * 32;      // pacc[(q·16 + i)·32 + c]
  double* dred = pacc + 4 * kDsmCS * 32; // [0]: gᵀd partial; [32..63]: backward scratch
  uint64_t* ibar = (uint64_t*)(dred + 64);
  uint64_t* vbar = ibar + 1;             // v_i arrived
  uint64_t* pbar = vbar + kDsmCS;        // partials of my q-th column arrived
  int* rdy = (int*)(pbar + 4);           // rdy[s]: my tile s is final (diagonal: W_j is ready)
  int* done = rdy + kD2Slots;            // done[s]: panels absorbed into my tile s
  int* list = done + kD2Slots;           // list[s] = (i << 8) | j
  int* pready = list + kD2Slots;         // P_j of my q-th column formed (chain CTAs)
  int* bcast = pready + 4;               // 2 per quad (test results, alternating)
  unsigned char* tslot = (unsigned char*)(bcast + 4);  // slot of tile (i, j) at [i·16 + j]
  cg::cluster_group cluster = cg::this_cluster();
  const int me = (int)cluster.block_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, quad = warp >> 2;
  const int t128 = tid & 127;
  const int NR = N + 1;
  const int ntc = (N + CHT - 1) / CHT, ntr = (NR + CHT - 1) / CHT;
  constexpr int NT = kDsmCS - NC;
  const bool chain = me < NC;
  int nchain = 0;  // my chain columns d2_col<NC>(me, 0 … nchain − 1), ascending (≤ 4 for NC ≥ 4)
  if (chain)
    while (nchain < 4 && d2_col<NC>(me, nchain) < ntc) ++nchain;
  const int jtop = nchain ? d2_col<NC>(me, nchain - 1) : -1;  // my highest chain column
  if (tid < 3 * kD2Slots + 8) rdy[tid] = 0;  // rdy, done, list, pready, bcast
  if (tid == 0) {
    dred[0] = 0.0;
    mbar_init(ibar, 1);
    for (int i = 0; i < kDsmCS; ++i) mbar_init(vbar + i, 1);
    for (int q = 0; q < 4; ++q) mbar_init(pbar + q, max(1, chain ? ntc - d2_col<NC>(me, q) - 3 : 1));
    fence_mbar_init();
  }
  for (int t = tid; t < 17 * 16; t += blockDim.x) {
    const int i = t >> 4, j = t & 15;
    if (j < ntc && i >= j && i < ntr) {
      const int s = d2_slot<NC>(i, j, ntr);
      tslot[t] = (unsigned char)s;
      if (d2_owner<NC>(i, j) == me) list[s] = (i << 8) | j;
    }
  }
  int nmine = 0;
  if (chain) {
    for (int q = 0; q < nchain; ++q) nmine += (d2_col<NC>(me, q) + 1 < ntr) ? 2 : 1;
  } else {
    for (int j = 0; j < ntc; ++j) nmine += d2_cntm(ntr - j - 2, ((me - NC - 3 * j) % NT + NT) % NT, NT);
  }
  __syncthreads();
  for (int s = warp; s < nmine; s += 8) {
    const int i = list[s] >> 8, j = list[s] & 255;
    const int r = CHT * i + lane, c0 = CHT * j;
    const bool rok = r < NR;
    double v[CHT];
#pragma unroll
    for (int c = 0; c < CHT; ++c) v[c] = (rok && c0 + c < N) ? __ldcg(M + r + (int64_t)(c0 + c) * ld) : 0.0;
    double* S = T + s * kTileD;
#pragma unroll
    for (int c = 0; c < CHT; ++c) S[lane * TLD + c] = v[c];
  }
  cluster.sync();  // flags and barriers initialised, every tile resident, cluster-wide
  if (me == 0 && tid == 0) D2STAMP(17, 0);

  auto qbar = [&]() { asm volatile("bar.sync %0, 128;" ::"r"(2 + quad) : "memory"); };
  auto rtile = [&](int i, int j) {
    return cluster.map_shared_rank(T, d2_owner<NC>(i, j)) + tslot[i * 16 + j] * kTileD;
  };
  auto rflag = [&](int i, int j) { return cluster.map_shared_rank(rdy, d2_owner<NC>(i, j)) + tslot[i * 16 + j]; };
  const int g = lane >> 2, t = lane & 3, qw = warp & 3;
  auto strip_af = [&](double* S, const double (&af)[8], const double* SB, double sgn, bool acc0) {
    double part[4][4][2];
#pragma unroll
    for (int h = 0; h < 4; ++h)
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) part[h][cb][0] = part[h][cb][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const double a = sgn * af[kk];
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) dmma(part[kk & 3][cb], a, SB[(8 * cb + g) * TLD + 4 * kk + t]);
    }
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double* dst = S + (8 * qw + g) * TLD + 8 * cb + 2 * t + e;
        const double base = acc0 ? *dst : 0.0;
        *dst = base + ((part[0][cb][e] + part[1][cb][e]) + (part[2][cb][e] + part[3][cb][e]));
      }
  };
  auto load_af = [&](const double* SA, double (&af)[8]) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) af[kk] = SA[(8 * qw + g) * TLD + 4 * kk + t];
  };
  auto copy_tile = [&](const double* src, double* dst) {
    double cp[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) cp[q] = (t128 + 128 * q < kTileD) ? src[t128 + 128 * q] : 0.0;
#pragma unroll
    for (int q = 0; q < 9; ++q)
      if (t128 + 128 * q < kTileD) dst[t128 + 128 * q] = cp[q];
  };

  int nab = 0;    // B-buffer parity
  int ntest = 0;  // bcast parity
  // Absorb panels done[s] … kmax into my tile s = (i, j).  For the last panel of a chain column
  // (k = j − 1) the operand L_{j,k} is the inbox; everything else is read from its owner.
  // Non-blocking: stop at the first panel whose operands are not published yet.
  auto absorb_upto = [&](int s, int i, int j, int kmax, bool blocking) {
    for (int k = done[s]; k <= kmax; ++k) {
      const bool inb = chain && k == j - 1;          // B (and A when i == j) from the inbox
      const int* fa = i == j ? nullptr : rflag(i, k);  // A = L_{i,k} (i > j: never the inbox)
      const int* fb = inb ? nullptr : rflag(j, k);
      const uint32_t ipar = (uint32_t)(d2_lc<NC>(j) - (me == 0)) & 1u;  // receptions before this one (CTA 0: none for column 0)
      if (blocking) {
        if (t128 == 0) {
          if (inb) d2_mbar_wait(ibar, ipar);
          if (fa)
            while (ld_acquire_cluster(fa) == 0) {
            }
          if (fb)
            while (ld_acquire_cluster(fb) == 0) {
            }
        }
        qbar();
      } else {
        int* bc = bcast + 2 * quad + (ntest++ & 1);
        if (t128 == 0) {
          bool ok = true;
          if (inb) ok = d2_mbar_test(ibar, ipar);
          if (ok && fa) ok = ld_acquire_cluster(fa) != 0;
          if (ok && fb) ok = ld_acquire_cluster(fb) != 0;
          *bc = ok;
        }
        qbar();
        if (!*bc) return;
      }
      const double* SB;
      if (inb) {
        SB = inbox;
      } else {
        double* B = Bq + (2 * quad + (nab++ & 1)) * kTileD;
        copy_tile(rtile(j, k), B);
        SB = B;
      }
      double af[8];
      if (i != j) load_af(rtile(i, k), af);
      if (!inb) qbar();
      if (i == j) load_af(SB, af);
      strip_af(T + s * kTileD, af, SB, -1.0, true);
      done[s] = k + 1;  // every thread writes its own copy of the same value
    }
  };
  auto finish = [&](int s, int i, int j) {
    double* S = T + s * kTileD;
    if (i == j) {
      qbar();  // every warp's rows of S are final
      const int c0 = CHT * j;
      diag_factor4(S, nullptr, 0, c0, min(CHT, N - c0), min(CHT, NR - c0), nullptr, Wb + d2_lc<NC>(j) * kTileD, info,
                   dscr, t128);
      if (t128 == 0) D2STAMP(j, 3);
      qbar();
      if (t128 == 0) st_release_cluster(rdy + s, 1);
      if (t128 == 0) D2STAMP(j, 1);
    } else if (chain) {  // (j + 1, j): W_j is local; push the result to the next chain CTA first
      if (t128 == 0)
        while (ld_acquire_cluster(rdy + 2 * d2_lc<NC>(j)) == 0) {
        }
      qbar();
      if (t128 == 0) D2STAMP(j, 4);
      double af[8];
      load_af(S, af);  // this warp's own rows
      strip_af(S, af, Wb + d2_lc<NC>(j) * kTileD, 1.0, false);
      fence_proxy_async();
      qbar();
      if (t128 == 0) D2STAMP(j, 6);
      if (t128 == 0) {
        if (i < ntc) {  // column i exists: its chain CTA absorbs L_{i,j} from its inbox
          const int c = i % NC;
          const uint32_t rb = d2_mapa(ibar, c);
          d2_remote_expect(rb, kD2Bytes);
          d2_push(d2_mapa(inbox, c), S, kD2Bytes, rb);
          d2_commit();
        }
        D2STAMP(j, 7);
        st_release_cluster(rdy + s, 1);
        D2STAMP(j, 2);
      }
    } else {
      const int od = j % NC;
      if (t128 == 0)
        while (ld_acquire_cluster(cluster.map_shared_rank(rdy, od) + 2 * d2_lc<NC>(j)) == 0) {
        }
      qbar();
      double* B = Bq + (2 * quad + (nab++ & 1)) * kTileD;
      copy_tile(cluster.map_shared_rank(Wb, od) + d2_lc<NC>(j) * kTileD, B);
      qbar();
      double af[8];
      load_af(S, af);
      strip_af(S, af, B, 1.0, false);
      qbar();
      if (t128 == 0) st_release_cluster(rdy + s, 1);
    }
  };

#pragma unroll 1
  for (int k = -1; k < ntc - 1; ++k) {
    for (int s = quad; s < nmine; s += 2) {
      const int i = list[s] >> 8, j = list[s] & 255;
      if (j == k + 1) {
        if (k >= 0) absorb_upto(s, i, j, k, true);
        if (i == j && t128 == 0) D2STAMP(j, 0);
      }
    }
    for (int s = quad; s < nmine; s += 2) {
      const int i = list[s] >> 8, j = list[s] & 255;
      if (j == k + 1) finish(s, i, j);
    }
    if (k >= 0)
      for (int s = quad; s < nmine; s += 2) {
        const int i = list[s] >> 8, j = list[s] & 255;
        if (j > k + 1) absorb_upto(s, i, j, k, false);
      }
  }
  __syncthreads();  // my tiles are final
  if (me == 0 && tid == 0) D2STAMP(17, 1);

  // ---- backward substitution v = L⁻ᵀ z ----
  const int rt = N / CHT, rrow = N % CHT;
  if (chain && warp >= 2 && warp < 6) {  // P_j = L_{j+1,j} W_j for my q-th column (q = warp − 2)
    const int q = warp - 2, j = q < nchain ? d2_col<NC>(me, nchain - 1 - q) : -1;
    if (jtop >= 0 && j >= 0 && j + 1 < ntc) {
      const double* L1 = T + (2 * d2_lc<NC>(j) + 1) * kTileD;
      const double* W = Wb + d2_lc<NC>(j) * kTileD;
      double* P = Bq + q * kTileD;
#pragma unroll 1
      for (int r = 0; r < CHT; ++r) P[r * TLD + lane] = d2_coldot(W, L1 + r * TLD, lane);  // Σ_s L1[r][s] W[s][c]
      __syncwarp();
      __threadfence_block();
      if (lane == 0) *(volatile int*)(pready + q) = 1;
    }
  }
  if (chain && warp == 0 && jtop >= 0) {  // v_j for my columns, descending
    double dp = 0.0;
    double* xb = dred + 32;
#pragma unroll 1
    for (int q = 0; q < nchain; ++q) {  // my columns, descending
      const int j = d2_col<NC>(me, nchain - 1 - q);
      const int* fz = rflag(rt, j);
      while (ld_acquire_cluster(fz) == 0) {
      }
      double acc = rtile(rt, j)[rrow * TLD + lane];  // z_j[c], c = lane
      const int np = ntc - j - 3;
      if (np > 0) {
        d2_mbar_wait(pbar + d2_lc<NC>(j), 0);
        for (int i = ntc - 1; i >= j + 3; --i) acc -= pacc[(d2_lc<NC>(j) * kDsmCS + i) * 32 + lane];
      }
      if (j + 2 < ntc) {
        const int* f2 = rflag(j + 2, j);
        while (ld_acquire_cluster(f2) == 0) {
        }
        const double* L2 = rtile(j + 2, j);
        double l2[CHT];
#pragma unroll
        for (int r = 0; r < CHT; ++r) l2[r] = L2[r * TLD + lane];
        d2_mbar_wait(vbar + j + 2, 0);
        const double* x = vin + (j + 2) * 32;
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int r = 0; r < CHT; ++r) s4[r & 3] = fma(l2[r], x[r], s4[r & 3]);
        acc -= (s4[0] + s4[1]) + (s4[2] + s4[3]);
      }
      xb[lane] = acc;
      __syncwarp();
      double v = d2_coldot(Wb + d2_lc<NC>(j) * kTileD, xb, lane);  // u_j = W_jᵀ acc
      if (j + 1 < ntc) {
        while (*(volatile int*)(pready + q) == 0) {
        }
        __threadfence_block();
        d2_mbar_wait(vbar + j + 1, 0);
        v -= d2_coldot(Bq + q * kTileD, vin + (j + 1) * 32, lane);  // P_jᵀ v_{j+1}
      }
      const int row = CHT * j + lane;
      v = row < N ? v : 0.0;
      vin[j * 32 + lane] = v;
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        D2STAMP(j, 5);
        for (int p = 1; p < kDsmCS; ++p) {  // the chain CTAs of j − 1, j − 2, j − 3 first, then the rest
          const int c = p < NC ? (me + NC - p) % NC : p;
          const uint32_t rb = d2_mapa(vbar + j, c);
          d2_remote_expect(rb, 256);
          d2_push(d2_mapa(vin + j * 32, c), vin + j * 32, 256, rb);
        }
        d2_commit();
        mbar_arrive(vbar + j);  // my own copy is in place
      }
      const double o = scale * v;
      if (row < N) {
        if (out) out[row] = o;
        if (dotv) dp += dotv[row] * o;
        if (yt) yt[row] = __dadd_rn(ybase[row], o);
      }
      __syncwarp();
    }
    dp = warp_allsum(dp);
    if (lane == 0) {
      dred[0] = dp;
      d2_wait_reads();
    }
  } else if (!chain && warp == 1) {  // partials L_ijᵀ v_i (i ≥ j + 3) for the chain CTA of j
    double* stage = dscr;
#pragma unroll 1
    for (int i = ntc - 1; i >= 3; --i) {
      bool any = false;
      for (int s = 0; s < nmine; ++s) any |= (list[s] >> 8) == i && (list[s] & 255) <= i - 3;
      if (!any) continue;
      d2_mbar_wait(vbar + i, 0);
      const double* x = vin + i * 32;
      for (int s = 0; s < nmine; ++s) {
        const int j = list[s] & 255;
        if ((list[s] >> 8) != i || j > i - 3) continue;
        stage[s * 32 + lane] = d2_coldot(T + s * kTileD, x, lane);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          const int c = j % NC, q = d2_lc<NC>(j);
          const uint32_t rb = d2_mapa(pbar + q, c);
          d2_remote_expect(rb, 256);
          d2_push(d2_mapa(pacc + (q * kDsmCS + i) * 32, c), stage + s * 32, 256, rb);
          d2_commit();
        }
      }
    }
    if (lane == 0) d2_wait_reads();
  }
  if (chain && quad == 1 && t128 == 0) d2_wait_reads();  // inbox pushes
  if (tid == 0)
    for (int i = 0; i < ntc; ++i) d2_mbar_wait(vbar + i, 0);  // every incoming copy has landed
  cluster.sync();  // all remote accesses done; dot partials ready
  if (me == 0 && tid == 0) D2STAMP(17, 2);
  if (me == 0 && tid == 0 && dot_out) {
    double sd = 0.0;
    for (int q = 0; q < NC; ++q) sd += cluster.map_shared_rank(dred, q)[0];
    *dot_out = sd;
  }
  cluster.sync();  // rank 0's reads complete before any CTA exits
}

template <int NC>
__global__ void __launch_bounds__(256, 1) k_chol_d2t(const double* __restrict__ M, int N, int ld,
                                                     double* __restrict__ out, double scale,
                                                     const double* __restrict__ dotv, double* dot_out, int* info,
                                                     const double* __restrict__ ybase, double* __restrict__ yt,
                                                     const DirGeo* geo, int want, int nmin, int nmax,
                                                     const CholArgs* ca) {
  chol_d2_body<NC>(M, N, ld, out, scale, dotv, dot_out, info, ybase, yt, geo, want, nmin, nmax, ca);
}
constexpr auto k_chol_d2 = k_chol_d2t<kD2Chain>;

// Graph mode: one node for both DSMEM-resident kernels, dispatching on the device geometry's N
// (k_chol_dsm for N ≤ 96, k_chol_d2 for 96 < N ≤ 512); dynamic shared memory kD2Smem.
template <int NC>
__global__ void __launch_bounds__(256, 1) k_chol_dsm_anyt(const double* __restrict__ M, double* __restrict__ out,
                                                         double scale, const double* __restrict__ dotv,
                                                         double* dot_out, int* info, const double* __restrict__ ybase,
                                                         double* __restrict__ yt, const DirGeo* geo, int want,
                                                         const CholArgs* ca) {
  if (geo->N <= kDsmUseMax)
    chol_dsm_body(M, 0, 0, out, scale, dotv, dot_out, info, ybase, yt, geo, want, kDsmUseMax, ca);
  else
    chol_d2_body<NC>(M, 0, 0, out, scale, dotv, dot_out, info, ybase, yt, geo, want, kDsmUseMax + 1, kDsmMaxN, ca);
}
constexpr auto k_chol_dsm_any = k_chol_dsm_anyt<kD2Chain>;

}  // namespace ssn
