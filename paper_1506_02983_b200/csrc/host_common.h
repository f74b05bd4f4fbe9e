// host_common.h -- host-side helpers shared by the single-GPU and the z-slab drivers (not ABI).
#pragma once
#include <algorithm>
#include <cmath>
#include "../../include/ecmg.h"
#include "ecmg_internal.cuh"

namespace ecmg {

inline LevelGeom make_geom(const ecmg_box& dom, const int n0[3], int k, const int face[6], int elem_path) {
  LevelGeom g{};
  for (int d = 0; d < 3; ++d) {
    g.n[d] = n0[d] << k;
    g.lo[d] = dom.lo[d];
    g.h[d] = (dom.hi[d] - dom.lo[d]) / g.n[d];
    const int lo = face[2 * d] == FACE_DIRICHLET ? 1 : 0;
    const int hi = face[2 * d + 1] == FACE_DIRICHLET ? g.n[d] - 1 : g.n[d];
    g.flo[d] = lo;
    g.nf[d] = std::max(0, hi - lo + 1);
  }
  g.P = ((long long)std::max(1, g.nf[0]) + 31) / 32 * 32;
  g.S = g.P * std::max(1, g.nf[1]);
  g.BP = ((long long)g.n[0] + 4 + 31) / 32 * 32;   // 256-B rows: TMA needs 16-B multiples
  g.BS = g.BP * (g.n[1] + 4);
  g.elem_path = elem_path;
  g.zoff = 0;
  g.zbeg = 0;
  g.zend = g.nf[2];
  g.nza = g.nf[2];
  g.zlo = 0;
  g.zhi = g.n[2] + 1;
  return g;
}

inline int beta_axes_w(const LevelGeom& g) { return std::max(g.n[0], std::max(g.n[1], g.n[2])) + 4; }
// the element-beta array (zero ring of 2) followed by the per-axis tables of beta_combine
inline long long beta_doubles(const LevelGeom& g) { return g.BS * (g.n[2] + 4) + beta_axes_doubles(beta_axes_w(g)); }
inline const double* beta_axes_ptr(const LevelGeom& g, const double* beta) { return beta + g.BS * (g.n[2] + 4); }
inline int beta_kind(int problem_id) {
  switch (problem_id) {
    case 3: return BETA_KIND_C3;
    case 5: return BETA_KIND_C5;
    case 22: return BETA_KIND_LAYERS;
    default: return BETA_KIND_ONE;
  }
}

inline ElemStencil make_elem_stencil(const LevelGeom& g, const Problem& pb, int precond) {
  ElemStencil es{};
  const double V = g.h[0] * g.h[1] * g.h[2];
  for (int pat = 0; pat < 8; ++pat) {
    double s = 0.0;
    for (int d = 0; d < 3; ++d) {
      double t = ((pat >> d) & 1) ? -1.0 : 1.0;
      t /= g.h[d] * g.h[d];
      for (int e = 0; e < 3; ++e)
        if (e != d) t *= ((pat >> e) & 1) ? (1.0 / 6.0) : (1.0 / 3.0);
      s += t;
    }
    es.kappa[pat] = V * s;
  }
  for (int F = 0; F < 6; ++F) {
    const int d = F >> 1;
    const int d1 = (d == 0) ? 1 : 0, d2 = (d == 2) ? 1 : 2;
    es.robin[F] = (pb.face[F] == FACE_ROBIN && pb.alpha[F] != 0.0) ? pb.alpha[F] * g.h[d1] * g.h[d2] : 0.0;
  }
  es.aq = (pb.id == PROB_ARRAYS) ? pb.arr[4] : nullptr;
  if (es.aq)   // alpha at the face Gauss points: every Robin face carries a mass term, its alpha read per element
    for (int F = 0; F < 6; ++F) {
      const int d = F >> 1, d1 = (d == 0) ? 1 : 0, d2 = (d == 2) ? 1 : 2;
      es.robin[F] = pb.face[F] == FACE_ROBIN ? g.h[d1] * g.h[d2] : 0.0;
    }
  es.precond = precond;
  es.cube = g.h[0] == g.h[1] && g.h[0] == g.h[2];
  es.bkind = -1;   // the caller enables beta on the fly (set_beta_fly) where the tables exist
  es.bw = 0;
  es.baxes = nullptr;
  return es;
}

inline ConstStencil make_const_stencil(const LevelGeom& g, double beta, int precond) {
  // c(o) = beta * sum_d K_d(o_d) prod_{e != d} M_e(o_e); K(0) = 2/h, K(1) = -1/h, M(0) = 2h/3, M(1) = h/6
  auto K = [](double h, int o) { return o ? -1.0 / h : 2.0 / h; };
  auto M = [](double h, int o) { return o ? h / 6.0 : 2.0 * h / 3.0; };
  auto c = [&](int ox, int oy, int oz) {
    const int o[3] = {ox, oy, oz};
    double s = 0.0;
    for (int d = 0; d < 3; ++d) {
      double t = K(g.h[d], o[d]);
      for (int e = 0; e < 3; ++e)
        if (e != d) t *= M(g.h[e], o[e]);
      s += t;
    }
    return beta * s;
  };
  ConstStencil cs{};
  for (int oz = 0; oz < 2; ++oz) {
    cs.c0[oz] = c(0, 0, oz);
    cs.cx[oz] = c(1, 0, oz);
    cs.cy[oz] = c(0, 1, oz);
    cs.cd[oz] = c(1, 1, oz);
  }
  cs.dinv = precond ? 1.0 / c(0, 0, 0) : 1.0;
  cs.diag = precond ? c(0, 0, 0) : 1.0;
  return cs;
}

inline int device_sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
      cudaGetLastError();
      sms = 148;
    }
  }
  return sms;
}

// planes per CTA (z chunk) of the JCG kernels
inline int auto_zc(int zchunk, int elem_path, const LevelGeom& g) {
  if (zchunk > 0) return zchunk;
  const int nz = g.zend - g.zbeg;
  const double slots = device_sm_count() * 2.0;   // both JCG kernels: 2 CTAs per SM (register bound)
  {
    // small levels (latency bound: a pass takes ~zc+2 dependent plane steps plus a fixed launch and
    // reduction cost): about 256 CTAs with chunks of >= 3 planes (tools/tune_zc_levels.py: 64^3 best at
    // zc 3-4, 128^3 at zc 8 (constant) / 16 (element), 20 % faster than 2 waves of 4-plane chunks)
    const double tiles = elem_path ? (double)((g.nf[0] + 31) / 32) * ((g.nf[1] + 15) / 16)
                                   : (double)((g.nf[0] + 31) / 32) * ((g.nf[1] + 31) / 32);
    if (tiles * (nz / 16) < 1.5 * slots) {
      long long nchunks = (long long)std::ceil(256.0 / tiles);
      nchunks = std::max(1LL, std::min(nchunks, (long long)std::max(1, nz / 3)));
      return (int)((nz + nchunks - 1) / nchunks);
    }
  }
  if (!elem_path) {   // constant stencil, 32 x 32 tiles: chunks of at most ~32 planes and at least 1.5 waves.
    // Measured (TMA loads without L2 promotion, tools/tune_elem.py --zc): 512^3 zc 171 (3 chunks, 2.6 waves)
    // 1.47 ms per iteration, zc 24-57 (8-22 waves) 1.36-1.41 ms; 256^3 zc 26 0.205 ms, zc 16-32 0.199 ms
    const long long tiles = (long long)((g.nf[0] + 31) / 32) * ((g.nf[1] + 31) / 32);
    const long long target = (long long)(device_sm_count() * 2 * 1.5);   // >= 1.5 waves
    long long nchunks = std::max((target + tiles - 1) / tiles, (long long)(nz + 31) / 32);
    nchunks = std::max(1LL, std::min(nchunks, (long long)std::max(1, nz / 4)));
    return (int)((nz + nchunks - 1) / nchunks);
  }
  // element path, 32 x 16 tiles, 2 CTAs per SM: the chunk count K maximising
  //   (fill of the last wave) x min(1, waves / 1.5) x zc / (zc + 2)
  // (a partial last wave idles SMs; fewer than ~1.5 waves cannot saturate HBM; every chunk re-reads
  // two halo planes). Measured on C3 256^3: the sweep is flat at the optimum and 10 % worse at 2.2 waves.
  // Chunks are capped at 64 planes: at 1024^3 (C5) the score above picks whole-z chunks (2048 CTAs,
  // zc 1023: 18.2 ms per iteration) while zc 32-64 measured 17.2-17.3 ms (tools/tune_elem.py --zc).
  const double tiles = (double)((g.nf[0] + 31) / 32) * ((g.nf[1] + 15) / 16);
  int best_zc = std::max(1, nz);
  double best = -1.0;
  for (int k = std::max(1, (nz + 63) / 64); k <= std::max(1, nz / 16); ++k) {
    const int zc = (nz + k - 1) / k;
    const int kk = (nz + zc - 1) / zc;
    const double waves = tiles * kk / slots;
    const double score = waves / std::ceil(waves) * std::min(1.0, waves / 1.5) * zc / (zc + 2.0);
    if (score > best + 1e-9) { best = score; best_zc = zc; }
  }
  return best_zc;
}


inline bool problem_faces(int id, int face[6], double alpha[6], int* nparams_required) {
  for (int f = 0; f < 6; ++f) { face[f] = FACE_DIRICHLET; alpha[f] = 0.0; }
  *nparams_required = 0;
  switch (id) {
    case 1: case 2: case 4: case 13: case 21: case 24: break;
    case 3: case 23: face[ZP] = FACE_ROBIN; alpha[ZP] = 1.0; break;
    case 25:   // Robin patch on the four side faces, a different alpha on each (face indexing pin)
      face[XM] = face[XP] = face[YM] = face[YP] = FACE_ROBIN;
      alpha[XM] = 2.0; alpha[XP] = 0.5; alpha[YM] = 1.5; alpha[YP] = 3.0;
      break;
    case 11: face[XP] = face[YP] = face[ZP] = FACE_ROBIN; break;   // Neumann (alpha = 0)
    case 12: face[XP] = face[YP] = FACE_ROBIN; break;
    case 5: *nparams_required = 48; break;
    case 22: *nparams_required = 15; break;
    default: return false;
  }
  return true;
}

inline long long free_count(const LevelGeom& g) { return (long long)g.nf[0] * g.nf[1] * (g.zend - g.zbeg); }
inline long long level_nodes(const LevelGeom& g) { return (long long)(g.n[0] + 1) * (g.n[1] + 1) * (g.n[2] + 1); }

// z-slab partition of a level with n cells along z over P ranks: the level is
// sharded iff n % (4P) == 0 and n / P >= 16 (every 4h EXP_finite block and 2h EXP_true cell then
// lies inside one slab, and each slab has >= 16 planes); rank r owns node planes
// [r n/P, (r+1) n/P), the last rank also plane n. Replicated levels: every rank owns [0, n+1).
inline bool& slab_force_single() {   // test only: shard even with P = 1 (single-rank NCCL self-test)
  static bool f = false;
  return f;
}

// min_n: levels with fewer z cells stay replicated even where they could be split (the driver's
// ECMG_OPT_SHARD_MIN: a split level pays two allreduces and two finalize launches per iteration)
inline bool slab_partition(int n, int P, int r, int* zlo, int* zhi, int min_n = 0) {
  const bool sharded = (P > 1 || slab_force_single()) && n % (4 * P) == 0 && n / P >= 16 && n >= min_n;
  if (!sharded) { *zlo = 0; *zhi = n + 1; return false; }
  *zlo = r * (n / P);
  *zhi = (r == P - 1) ? n + 1 : (r + 1) * (n / P);
  return true;
}

// geometry of rank r's slab of a level (work vectors: owned free planes + one halo plane per side)
inline LevelGeom slab_geom(LevelGeom g, int P, int r, bool* sharded, int min_n = 0) {
  int zlo, zhi;
  *sharded = slab_partition(g.n[2], P, r, &zlo, &zhi, min_n);
  if (!*sharded) return g;
  g.zlo = zlo;
  g.zhi = zhi;
  const int f0 = g.flo[2], f1 = g.flo[2] + g.nf[2];            // global free node planes [f0, f1)
  const int a = std::max(zlo, f0), b = std::min(zhi, f1);       // owned free planes [a, b)
  g.zoff = a - f0 - 1;                                          // local plane 0 = free plane a-1 (halo)
  g.zbeg = 1;
  g.zend = 1 + std::max(0, b - a);
  g.nza = g.zend + 1;
  return g;
}

}  // namespace ecmg

namespace ecmg {
// element kernels form beta from the level's axis tables (analytic beta) instead of reading the array
inline void set_beta_fly(ElemStencil& es, const LevelGeom& g, const Problem& pb, const double* beta) {
  if (pb.id == PROB_ARRAYS) return;   // caller beta: no analytic axis tables, the kernels read the array
  es.bkind = beta_kind(pb.id);
  es.bw = beta_axes_w(g);
  es.baxes = beta_axes_ptr(g, beta);
}
}  // namespace ecmg
