// K4, DSMEM-resident form (N ≤ 512, the hot path's Eq. (18) / (19) systems at m ≤ 512): the
// Cholesky factor of the N × N SPD matrix, the forward substitution (the right-hand side carried as
// row N) and the backward substitution, by one 16-CTA thread-block cluster whose distributed
// shared memory holds the whole lower triangle.  CTA j owns block column j (32 columns): its row
// tiles (i, j), i = j … ⌈(N+1)/32⌉ − 1, live in its shared memory for the whole launch (≤ 17 × 8.4
// KB), so no tile ever makes a round trip through L2.
//
// Right-looking by panels, left-looking per owner.  CTA j absorbs panel k < j (tile update
// A_ij −= L_ik L_jkᵀ, DMMA) as soon as CTA k has published the tiles it needs, reading L_ik straight
// from CTA k's shared memory; then it factors its diagonal tile (diag_factor4: L_jj and W_j =
// L_jj⁻¹), forms L_ij = A_ij W_jᵀ for its other tiles (DMMA) and publishes each one with a
// release store of a per-tile flag in its own shared memory (consumers poll it with cluster-scope
// acquire loads).  Two 128-thread quads split an owner's tiles by parity (quad 0: the diagonal and
// even offsets; quad 1: odd offsets, so tile (j+1, j) — the next owner's critical input — is
// quad 1's first).  The backward solve v = L⁻ᵀz is a chain over the owners (j = last … 0), each
// waiting for v_i of the owners i > j (release/acquire flag again).  The outputs are those of
// k_chol_cluster: out = scale·v, *dot_out = Σ dotv·out, yt = ybase + out, *info = 1 on a
// non-positive pivot.  The factor itself is not written back to M (the hot path does not reuse it).
#pragma once
#include <cooperative_groups.h>
#include "k_newton.cuh"

namespace ssn {

constexpr int kDsmCS = 16;  // cluster size = max block columns (N ≤ 512)
constexpr int kDsmUseMax = 96;  // k_chol_dsm for N ≤ 96 (faster there than k_chol_d2: N = 64 20.7 vs 22.7 µs)
constexpr int kDsmMaxN = kDsmCS * CHT;     // 512
constexpr int kDsmTiles = kDsmCS + 1;      // row tiles of column 0 at N = 512 (NR = 513)
constexpr int kTileD = CHT * TLD;          // doubles per smem tile (32 × 33)
constexpr size_t kDsmSmemDoubles =
    (size_t)kDsmTiles * kTileD + 2 * kTileD + kTileD + kDiagScratch + kDsmCS * 32 + 32 + 64;
constexpr size_t kDsmSmem = kDsmSmemDoubles * sizeof(double);

#ifdef DSM_PROBE
__device__ unsigned long long g_dsm[kDsmCS][16];
#define DSTAMP(i) do { if ((tid & 127) == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_dsm[j][i] = t_; } } while (0)
#define DCLK(i) do { if ((tid & 127) == 0) g_dsm[j][i] = clock64(); } while (0)
#else
#define DCLK(i) do {} while (0)
#define DSTAMP(i) do {} while (0)
#endif

SSN_DEV int ld_acquire_cluster(const int* p) {
  int v;
  asm volatile("ld.acquire.cluster.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SSN_DEV void st_release_cluster(int* p, int v) {
  asm volatile("st.release.cluster.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
SSN_DEV void red_release_cluster_add(int* p, int v) {
  asm volatile("red.release.cluster.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

SSN_DEV void chol_dsm_body(const double* __restrict__ M, int N, int ld, double* __restrict__ out, double scale,
                           const double* __restrict__ dotv, double* dot_out, int* info,
                           const double* __restrict__ ybase, double* __restrict__ yt, const DirGeo* geo, int want,
                           int nmax, const CholArgs* ca) {
  namespace cg = cooperative_groups;
  if (geo) {  // graph mode: predicated on the branch and on N ≤ nmax ≤ 512 (uniform over the cluster)
    if ((want >= 0 ? geo->branch != want : (geo->branch != 1 && geo->branch != 2)) || geo->N > nmax) return;
    if (ca) {  // want < 0: the outputs of whichever exact branch this step took
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
  extern __shared__ double sm[];
  double* T = sm;                          // T + s·kTileD = tile (j + s, j), row-major, TLD
  double* Bq = T + kDsmTiles * kTileD;     // per quad: local copy of L_jk for the current panel
  double* Wj = Bq + 2 * kTileD;            // W_j = L_jj⁻¹ (row-major, TLD)
  double* dscr = Wj + kTileD;              // diag_factor4 scratch
  double* vin = dscr + kDiagScratch;       // vin[i][·] = v_i, pushed by owner i > j (backward)
  double* dred = vin + kDsmCS * 32;        // gᵀd partial
  int* ready = (int*)(dred + 32);          // ready[s]: tile (j + s, j) holds L (s ≥ 1)
  int* vflag = ready + kDsmTiles;          // vflag[i] = 32 once vin[i] has arrived
  int* wready = vflag + kDsmCS;            // W_j ready (quad 0 → quad 1, local)
  int* upd = wready + 1;                   // upd[s]: panels absorbed into tile s (quad 1 → TRSMs, local)
  int* tnext = upd + kDsmTiles;            // TRSM work counter, and one broadcast slot per quad
  int* bcast = tnext + 1;
  constexpr int kFlags = kDsmTiles + kDsmCS + 1 + kDsmTiles + 1 + 2;
  cg::cluster_group cluster = cg::this_cluster();
  const int j = (int)cluster.block_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, quad = warp >> 2, qw = warp & 3;
  const int t128 = tid & 127, g = lane >> 2, t = lane & 3;
  const int NR = N + 1;
  const int ntc = (N + CHT - 1) / CHT, ntr = (NR + CHT - 1) / CHT;
  const bool own = j < ntc;
  const int nt = own ? ntr - j : 0;  // my tiles
  const int c0 = CHT * j;
  if (tid == 0) DSTAMP(0);
  if (tid < kFlags) ready[tid] = 0;
  // load my block column: tile (i, j) rows [32i, 32i+32) ∩ [0, NR), cols [32j, 32j+32) ∩ [0, N)
  for (int s = warp; s < nt; s += 8) {
    const int r = CHT * (j + s) + lane;
    const bool rok = r < NR;
    double v[CHT];
#pragma unroll
    for (int c = 0; c < CHT; ++c) v[c] = (rok && c0 + c < N) ? __ldcg(M + r + (int64_t)(c0 + c) * ld) : 0.0;
    double* S = T + s * kTileD;
#pragma unroll
    for (int c = 0; c < CHT; ++c) S[lane * TLD + c] = v[c];
  }
  cluster.sync();  // flags initialised and every column resident, cluster-wide
  if (tid == 0) DSTAMP(1);

  auto qbar = [&]() { asm volatile("bar.sync %0, 128;" ::"r"(2 + quad) : "memory"); };
  // publish: the quad's shared-memory writes are ordered before the flag by the barrier and the
  // release store's cumulativity
  auto qrelease = [&](int* f) {
    qbar();
    if (t128 == 0) st_release_cluster(f, 1);
  };
  auto lwait = [&](const int* f, int v) {  // local flag (volatile poll by one thread)
    if (t128 == 0)
      while (*(volatile const int*)f < v) __nanosleep(32);
    qbar();
  };
  auto lpost = [&](int* f, int v) {
    __threadfence_block();
    qbar();
    if (t128 == 0) *(volatile int*)f = v;
  };
  // Watermark over CTA k's ready flags: the number w ≥ need of consecutive published tiles
  // (k + s0 + q, k), q = 0, 1, …, read in one round trip (lane q polls flag s0 + q).
  auto watermark = [&](const int* rk, int s0, int cnt, int need) {
    if (qw == 0) {
      int w = 0;
      for (;;) {
        const bool f = lane < cnt && ld_acquire_cluster(rk + s0 + lane) != 0;
        const unsigned b = __ballot_sync(0xffffffffu, f);
        w = __ffs(~b) - 1;
        if (b == 0xffffffffu) w = 32;
        if (w > cnt) w = cnt;
        if (w >= need) break;
        __nanosleep(64);
      }
      if (lane == 0) bcast[quad] = w;
    }
    qbar();
    const int w = bcast[quad];
    qbar();
    return w;
  };
  // rows 8qw … 8qw+7 of tile S: S = (acc0 ? S : 0) + sgn · A · SBᵀ, with this warp's A fragments
  // af[kk] = A[8qw + g][4kk + t] already in registers (32 × 32 × 32, DMMA, 4 accumulator groups)
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

  if (own) {
    double* Bmy = Bq + quad * kTileD;
    // Quad 0 carries the critical chain: the diagonal tile and tile (j+1, j) absorb the panels
    // k < j, then L_jj, W_j and L_{j+1,j} (the next owner's input) at once.  Quad 1 absorbs the
    // panels into the tiles s ≥ 2 (panel by panel, ascending s; remote operands prefetched one
    // tile ahead) and counts them in upd[].  Then both take L_ij = A_ij W_jᵀ for s ≥ 2 in
    // ascending s from a shared counter, each tile once it has absorbed every panel.
    const int q0n = nt > 1 ? 2 : 1;  // quad 0's tiles: s = 0 (and 1)
#pragma unroll 1
    for (int k = 0; k < (quad == 0 || nt > 2 ? j : 0); ++k) {
      const double* Tk = cluster.map_shared_rank(T, k);
      const int* rk = cluster.map_shared_rank(ready, k);
      // quad 0: L_jk (and L_{j+1,k}); quad 1: L_jk and its operand tiles s ≥ 2 as published
      int w = watermark(rk, j - k, quad == 0 ? q0n : nt, quad == 0 ? q0n : min(3, nt));
      const double* Ljk = Tk + (j - k) * kTileD;
      double cp[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) cp[q] = (t128 + 128 * q < kTileD) ? Ljk[t128 + 128 * q] : 0.0;
#pragma unroll
      for (int q = 0; q < 9; ++q)
        if (t128 + 128 * q < kTileD) Bmy[t128 + 128 * q] = cp[q];
      if (quad == 0) {
        double af[8], a1[8];
        if (nt > 1) load_af(Tk + (j + 1 - k) * kTileD, a1);
        qbar();
        load_af(Bmy, af);
        strip_af(T, af, Bmy, -1.0, true);
        if (nt > 1) strip_af(T + kTileD, a1, Bmy, -1.0, true);
      } else {
        double af[8], an[8];
        load_af(Tk + (j + 2 - k) * kTileD, an);  // w ≥ 3: tile (j+2, k) is published
        qbar();
#pragma unroll 1
        for (int s = 2; s < nt; ++s) {
#pragma unroll
          for (int q = 0; q < 8; ++q) af[q] = an[q];
          if (s + 1 < nt) {
            if (s + 1 >= w) w = watermark(rk, j - k, nt, s + 2);
            load_af(Tk + (j + s + 1 - k) * kTileD, an);
          }
          strip_af(T + s * kTileD, af, Bmy, -1.0, true);
          lpost(upd + s, k + 1);
        }
      }
      qbar();  // Bmy is rewritten by the next panel
    }
    if (quad == 0) DSTAMP(2); else DSTAMP(8);
    if (quad == 0) {
      diag_factor4(T, nullptr, 0, c0, min(CHT, N - c0), min(CHT, NR - c0), nullptr, Wj, info, dscr, t128);
      lpost(wready, 1);
      DSTAMP(3);
      if (nt > 1) {  // L_{j+1,j} first: the next owner's critical input
        double af[8];
        load_af(T + kTileD, af);
        strip_af(T + kTileD, af, Wj, 1.0, false);
        qrelease(ready + 1);
        DSTAMP(4);
      }
    } else {
      lwait(wready, 1);
    }
#pragma unroll 1
    for (;;) {
      if (t128 == 0) bcast[quad] = atomicAdd(tnext, 1) + 2;
      qbar();
      const int s = bcast[quad];
      qbar();
      if (s >= nt) break;
      lwait(upd + s, j);
      double af[8];
      load_af(T + s * kTileD, af);
      strip_af(T + s * kTileD, af, Wj, 1.0, false);
      qrelease(ready + s);
    }
    if (quad == 0) DSTAMP(5); else DSTAMP(9);
  }
  __syncthreads();
  // ---- backward substitution v = L⁻ᵀ z, z = row N of the factor (forward substitution) ----
  // Owner j waits for v_i (i > j, pushed into its vin[i] by owner i; 32 per-lane release
  // increments of vflag[i]) in descending i, then pushes v_j to every owner c < j.
  if (own && warp == 0) {
    const int rt = N / CHT, rrow = N % CHT;
    double acc = T[(rt - j) * kTileD + rrow * TLD + lane];  // z_j[c], c = lane
#pragma unroll 1
    for (int i = ntc - 1; i > j; --i) {
      while (ld_acquire_cluster(vflag + i) < 32) {
      }
      const double vi = vin[i * 32 + lane];  // v_i[r], r = lane
      const double* Lij = T + (i - j) * kTileD;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int r = 0; r < CHT; r += 2) {  // Σ_r L_ij[r][c] v_i[r]
        s0 = fma(Lij[r * TLD + lane], __shfl_sync(0xffffffffu, vi, r), s0);
        s1 = fma(Lij[(r + 1) * TLD + lane], __shfl_sync(0xffffffffu, vi, r + 1), s1);
      }
      acc -= s0 + s1;
    }
    double v0 = 0.0, v1 = 0.0;  // v_j[c] = Σ_r W_j[r][c] z_j[r]
#pragma unroll
    for (int r = 0; r < CHT; r += 2) {
      v0 = fma(Wj[r * TLD + lane], __shfl_sync(0xffffffffu, acc, r), v0);
      v1 = fma(Wj[(r + 1) * TLD + lane], __shfl_sync(0xffffffffu, acc, r + 1), v1);
    }
    const int row = c0 + lane;
    const double v = row < N ? v0 + v1 : 0.0;
    for (int c = j - 1; c >= 0; --c) {  // nearest consumer first: it is next on the chain
      cluster.map_shared_rank(vin, c)[j * 32 + lane] = v;
      red_release_cluster_add(cluster.map_shared_rank(vflag, c) + j, 1);
    }
    if (lane == 0) DSTAMP(6);
    const double o = scale * v;
    double dp = 0.0;
    if (row < N) {
      if (out) out[row] = o;
      if (dotv) dp = dotv[row] * o;
      if (yt) yt[row] = __dadd_rn(ybase[row], o);
    }
    dp = warp_allsum(dp);
    if (lane == 0) dred[0] = dp;
  }
  cluster.sync();  // all remote accesses done; dot partials ready
  if (j == 0 && tid == 0 && dot_out) {
    double sd = 0.0;
    for (int q = 0; q < ntc; ++q) sd += cluster.map_shared_rank(dred, q)[0];
    *dot_out = sd;
  }
  cluster.sync();  // rank 0's reads complete before any CTA exits
  if (tid == 0) DSTAMP(7);
}

__global__ void __launch_bounds__(256, 1) k_chol_dsm(const double* __restrict__ M, int N, int ld,
                                                     double* __restrict__ out, double scale,
                                                     const double* __restrict__ dotv, double* dot_out, int* info,
                                                     const double* __restrict__ ybase, double* __restrict__ yt,
                                                     const DirGeo* geo, int want, int nmax, const CholArgs* ca) {
  chol_dsm_body(M, N, ld, out, scale, dotv, dot_out, info, ybase, yt, geo, want, nmax, ca);
}

}  // namespace ssn
