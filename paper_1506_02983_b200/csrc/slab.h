// slab.h -- z-slab driver interface (ecmg_slab.cu), used by ecmg_api.cu. Not part of the ABI.
#pragma once
#include <vector>
#include "../../include/ecmg.h"
#include "ecmg_internal.cuh"

namespace ecmg {

struct SlabCfg {
  ecmg_box dom;
  int n0[3];
  int L;
  Problem prob;
  int elem_path, exp_variant, precond, kernel_variant, zchunk;
  int fused_halo;   // 1: K2 / init store their boundary planes into the neighbours' halo planes
  int beta_fly;     // 1: element kernels form analytic beta from the level's axis tables
  int shard_min;    // levels with fewer z cells are replicated (ECMG_OPT_SHARD_MIN)
  int use_graph;    // 1: tolerance-stopped solves of sharded levels run as one CUDA graph per level with a
                    // device-set WHILE node (ECMG_OPT_GRAPH); 0: the host loop with batched readbacks
  // ECMG_PROB_ARRAYS: the caller's device arrays, 5 per level (beta_e, f_q, g_D, g_R, alpha_q), global-domain
  // layouts (every slab reads its planes by global index); empty for the registry problems
  std::vector<const double*> arrays;
};
constexpr int kShardMinDefault = 256;

struct SlabDriver;
// P slabs; virt = all P in this process on one GPU (test fixture), else this process is `rank` of P
// NCCL ranks (nccl_id: the 128-byte ncclUniqueId). *status receives the ecmg_status.
SlabDriver* slab_driver_create(const SlabCfg& cfg, int P, int rank, bool virt, const unsigned char* nccl_id, int* status);
void slab_driver_configure(SlabDriver* d, const SlabCfg& cfg);
void slab_driver_destroy(SlabDriver* d);
// levels [k_begin, L) (levels below k_begin: u_k imported with slab_import_u, per_level left untouched)
int slab_run(SlabDriver* d, double eps, ecmg_stats* per_level, double* u_out, bool u_dev, double* ut_out, bool ut_dev,
             cudaStream_t stream, int k_begin);
// the finest level's setup on the driver's own low-priority stream (forked from `stream`); the next
// slab_run waits for it instead of setting the finest level up in line
int slab_setup_ahead(SlabDriver* d, cudaStream_t stream);
// first sharded level (L if none); every level below it is replicated
int slab_first_sharded(const SlabDriver* d);
// copy a full-layout level-k solution into every local slab's u_k (the replicated levels' solutions)
int slab_import_u(SlabDriver* d, int k, const double* u_full, cudaStream_t stream);
int slab_solve_level(SlabDriver* d, int k, double eps, int max_iter, double* u, ecmg_stats* st, cudaStream_t stream);
void slab_level_range(const SlabDriver* d, int k, int* zlo, int* zhi);
void slab_last_timing(const SlabDriver* d, double* ms, int* it, long long* nfree);
int nccl_unique_id(unsigned char id[128]);

}  // namespace ecmg
