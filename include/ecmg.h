/*
 * ecmg.h -- C ABI of libecmg, the B200-native hot path of ECMG_jcg (Pan, He, Hu,
 * "A new extrapolation cascadic multigrid method for 3D elliptic boundary value problems",
 * arXiv:1506.02983). "P:n" cites /root/reference/PAPER.md line n; section / equation labels
 * are the LaTeX \label names of the paper.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Every function returns ECMG_OK (0) or a negative ecmg_status; none throws or aborts.
 *  - A grid is bound to one CUDA device and one CUDA stream (given at creation). All device work
 *    of a call is enqueued on that stream; a call returns after its results are complete
 *    (calls synchronise the stream before returning, so host-visible outputs are valid).
 *  - Nodal vectors passed by the caller are contiguous fp64 arrays over all (nx+1)(ny+1)(nz+1)
 *    nodes of the level, x fastest: index ix + (nx+1)(iy + (ny+1) iz).
 *    Device pointers are required except where a parameter says "device or host".
 *    The caller owns them; the library reads / writes them only during the call.
 *  - The grid owns all internal workspace (pitched free-box vectors, element coefficients,
 *    reduction buffers). Nothing the caller passes is retained after a call returns, with ONE
 *    exception: the per-level device arrays of ECMG_PROB_ARRAYS (ecmg_problem.level_arrays), which
 *    the grid keeps from ecmg_set_coeffs until the next ecmg_set_coeffs or ecmg_destroy_grid.
 *  - There is no CPU fallback: without a usable CUDA device ecmg_create_grid fails with
 *    ECMG_ECUDA.
 *  - A grid is not thread safe; distinct grids may be used from distinct threads.
 */
#ifndef ECMG_H
#define ECMG_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ECMG_OK = 0,
  ECMG_EINVAL = -1,      /* bad argument (sizes, pointers, problem parameters, beta <= 0, alpha < 0) */
  ECMG_ENOMEM = -2,      /* device allocation failed */
  ECMG_ENOTCONV = -3,    /* relative-residual tolerance not met within max_iter (stats still filled) */
  ECMG_EBREAKDOWN = -4,  /* p.Ap <= 0 inside JCG: the operator is not SPD */
  ECMG_EDIAG = -5,       /* non-positive diagonal entry: Jacobi preconditioner undefined */
  ECMG_EMISMATCH = -6,   /* level index / grid embedding mismatch */
  ECMG_ECUDA = -7,       /* CUDA runtime error or no device */
  ECMG_ENCCL = -8        /* NCCL error (multi-GPU z-slabs) */
} ecmg_status;

/* Boundary kinds of Eq. (bvp). Robin with alpha = 0 is Neumann. */
typedef enum { ECMG_DIRICHLET = 0, ECMG_ROBIN = 1 } ecmg_face_kind;

/* Built-in problems (device-side registry; beta, f, g_D, alpha, g_R as functions of x).
 * C1..C5 are BASELINE.json configs[0..4]; P1..P3 are the paper's Problems 1-3;
 * PATCH_* are Galerkin-exact patch tests; CONST_F is f = 1 with homogeneous Dirichlet. */
typedef enum {
  ECMG_PROB_C1 = 1,   /* beta=1, u=sin(pi x)sin(pi y)sin(pi z), Dirichlet all faces */
  ECMG_PROB_C2 = 2,   /* beta=1, u=exp(x+y+z), Dirichlet all faces */
  ECMG_PROB_C3 = 3,   /* beta=1+sin(2pi x)cos(2pi y)sin(2pi z)/2, u=cos(pi x)cos(pi y)e^z, Robin z=1 (alpha=1) */
  ECMG_PROB_C4 = 4,   /* beta=1, u=(x^2+y^2+z^2)^(3/4), Dirichlet all faces */
  ECMG_PROB_C5 = 5,   /* layered geology: params[48] (layout in synth/__init__.py), f Gaussian, g_D=0 */
  ECMG_PROB_P1 = 11,  /* paper Problem 1: Neumann on x=1,y=1,z=1 */
  ECMG_PROB_P2 = 12,  /* paper Problem 2: Neumann on x=1,y=1 */
  ECMG_PROB_P3 = 13,  /* paper Problem 3: singular, Dirichlet all faces */
  ECMG_PROB_PATCH_TRILINEAR = 21,
  ECMG_PROB_PATCH_LAYERED = 22, /* params[15]: the C5 layer set */
  ECMG_PROB_PATCH_ROBIN = 23,
  ECMG_PROB_CONST_F = 24,
  ECMG_PROB_PATCH_ROBIN_XY = 25, /* linear patch, Robin on x-, x+, y-, y+ with alpha 2, 0.5, 1.5, 3 */
  ECMG_PROB_ARRAYS = 100  /* the caller's data per level (ecmg_problem.level_arrays), any face kinds */
} ecmg_problem_id;

typedef struct { double lo[3], hi[3]; } ecmg_box;  /* domain Omega = [lo, hi]; hi > lo */

/* Multi-GPU z-slab decomposition (NULL or nranks == 1: single GPU). nccl_id is the 128-byte
 * ncclUniqueId that rank 0 created and the caller broadcast (e.g. with torch.distributed). */
typedef struct { int rank, nranks; unsigned char nccl_id[128]; } ecmg_dist;

typedef struct ecmg_grid ecmg_grid;  /* opaque; owns all internal workspace */

/* Build the embedded grid hierarchy of Alg. 4: level k has coarsest_cells[d] * 2^k
 * cells along axis d, k = 0 .. num_levels-1; the finest mesh size is H / 2^(num_levels-1)
 * (P:287-288 with L = num_levels - 2). Levels 0 and 1 are the DSOLVE levels.
 *   dom            domain box, extents > 0
 *   coarsest_cells >= 1 per axis (>= 2 recommended)
 *   num_levels     >= 3 (two DSOLVE levels + at least one ECMG level)
 *   dist           NULL for a single GPU
 *   cuda_stream    cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); NULL = default stream
 *   out            receives the grid; *out is NULL on failure
 * Errors: ECMG_EINVAL, ECMG_ECUDA (no device), ECMG_ENOMEM (workspace for the finest level). */
int ecmg_create_grid(const ecmg_box* dom, const int coarsest_cells[3], int num_levels,
                     const ecmg_dist* dist, void* cuda_stream, ecmg_grid** out);

typedef struct {
  ecmg_face_kind face[6];   /* x-, x+, y-, y+, z-, z+; must equal the problem's own boundary kinds */
  int problem_id;           /* ecmg_problem_id */
  const double* params;     /* host array, problem parameters (C5: 48 doubles, PATCH_LAYERED: 15,
                               ARRAYS: 6 = alpha per face, read on Robin faces, >= 0; a spatially varying
                               alpha is given at the face Gauss points through level_arrays
                               [4L+k], below). Copied. */
  int n_params;
  /* ECMG_PROB_ARRAYS only (else NULL / 0): n_level_arrays = 4 * num_levels device pointers, level k's
   * data of Eq. (bvp) at the points the discretisation reads:
   *   [4k+0] beta_e   n_x n_y n_z doubles, element e = ex + n_x (ey + n_y ez); beta > 0 (not checked);
   *                   NULL on every level = beta 1 (then all-Dirichlet problems take the constant stencil)
   *   [4k+1] f_q      8 per element, index 8 e + q, q = q_x + 2 q_y + 4 q_z: the 2x2x2 Gauss point
   *                   lo + (e + (1 +- 1/sqrt(3)) / 2) h per axis, bit set = the + point; NULL = f 0
   *   [4k+2] gD       (n_x+1)(n_y+1)(n_z+1) nodes, x fastest, read on Dirichlet nodes only; NULL = 0
   *   [4k+3] gR       per face F = x-, x+, y-, y+, z-, z+ a block of 4 n_d1 n_d2 values (d1 < d2 the in-face
   *                   axes), index 4 (e1 + n_d1 e2) + q, q = q_1 + 2 q_2 the 2x2 face Gauss point; read on
   *                   Robin faces only; NULL = 0
   * n_level_arrays = 5 * num_levels adds, after those 4 * num_levels pointers, one per level:
   *   [4L+k] alpha_q  alpha at the 2x2 face Gauss points, gR's layout and points (Eq. bvp's piecewise smooth
   *                   alpha), read on Robin faces only, >= 0 (not checked); NULL on a level = the
   *                   per-face alpha of params on that level. The Robin face mass of a face element is then
   *                   h1 h2 / 4 sum_q alpha_q N_c(q) N_d(q), the 2x2 rule the Robin load uses.
   * The grid keeps the pointers: the arrays are read by every call that runs a level's setup, a Dirichlet
   * fill or the operator (ecmg_run, ecmg_run_fixed, ecmg_solve_level, ecmg_level_rhs, ecmg_apply_operator, the
   * EXP calls) and must stay valid and unchanged until the next ecmg_set_coeffs or ecmg_destroy_grid (DESIGN.md
   * reading R6).
   * On z-slabs (NCCL ranks or virtual slabs) every rank passes the global-domain arrays in its own device
   * memory; each rank reads its planes by global index. */
  const double* const* level_arrays;
  int n_level_arrays;
} ecmg_problem;

/* Bind the problem of Eq. (bvp) to the grid. Level operators are matrix-free; the
 * per-level setup (element beta at centroids, 2x2x2-Gauss load, 2x2-Gauss Robin terms, Dirichlet
 * lifting, ||f_h||) runs inside ecmg_solve_level / ecmg_run (it is part of the timed hot path).
 * Errors: ECMG_EINVAL (unknown id, wrong n_params, face kinds differ from the problem's,
 * beta <= 0 or alpha < 0 in the parameters). */
int ecmg_set_coeffs(ecmg_grid* grid, const ecmg_problem* problem);

typedef enum {
  ECMG_OPT_EXP_VARIANT = 1,  /* 0 (default): 20-node Serendipity EXP_finite;
                                1: Remark 2's 27-node tri-quadratic Lagrange */
  ECMG_OPT_PRECOND = 2,      /* 1 (default): Jacobi, ECMG_jcg; 0: plain CG, ECMG_cg */
  ECMG_OPT_ZCHUNK = 3,       /* planes per CTA in the z-marching JCG kernels (tuning; 0 = auto) */
  ECMG_OPT_KERNEL = 4,       /* constant-coefficient JCG kernels: 1 (default) TMA-fed smem ring,
                                0 register-prefetch loads (ablation) */
  ECMG_OPT_GRAPH = 5,        /* tolerance-stopped JCG loop: 1 (default) one CUDA graph per level with a
                                device-set conditional WHILE node (z-slab split levels too: the allreduces
                                and halo exchanges are captured into the WHILE body; if capture fails the
                                slab driver falls back to the host loop); 0 host loop with batched readbacks */
  ECMG_OPT_PERSISTENT = 7,   /* levels with at most this many free unknowns (and at most 4 bricks of
                                8x8x4 nodes per resident CTA) run the whole JCG solve in one cooperative
                                launch with the nodes' values in registers, both operators (default
                                40000, i.e. up to 32^3 cells; 0 = off; larger levels up to
                                ECMG_OPT_PERS_TMA take the cooperative TMA solve: measured 64^3 0.82 ->
                                0.67 ms on C4) */
  ECMG_OPT_PDL = 8,          /* 1: the JCG kernels use programmatic dependent launch (the next kernel's
                                launch overlaps the previous one's tail); 0 (default): plain launches
                                (measured on B200: no difference inside the per-level CUDA graphs) */
  ECMG_OPT_FUSED_HALO = 9,   /* z-slabs: 1 (default) the K2 / init passes store their boundary planes of
                                the vector the next K1 reads straight into the neighbours' halo planes
                                (another slab on this GPU, or the neighbour rank's buffer mapped with
                                CUDA IPC over NVLink; ranks fall back to 0 together if any mapping
                                fails); 0: halo planes by device copy / ncclSend-ncclRecv */
  ECMG_OPT_SETUP_AHEAD = 10, /* ecmg_run / ecmg_run_fixed: 1 (default) every level's setup (element beta,
                                lifted right-hand side, g_D on the Dirichlet nodes of u_k; row a1 depends
                                on no solution) is enqueued up front on a low-priority internal stream and
                                overlaps the latency-bound coarse solves, which run on a high-priority
                                internal stream (both forked from and joined back into the grid's stream);
                                0: each level's setup runs in line before its solve */
  ECMG_OPT_EXP_KERNEL = 12,  /* EXP_finite: 1 (default) one fused pass (seeds formed per 4h layer in shared
                                memory, fine level written once); 0: seed pass + interpolation pass
                                (ablation; bitwise the same results) */
  ECMG_OPT_CTA_SOLVE = 13,   /* levels with at most this many free unknowns (default 1000, at most 4096)
                                are solved by ONE CTA with every vector in shared memory (no grid barrier);
                                0: off (the cooperative persistent kernel takes them) */
  ECMG_OPT_PERS_TMA = 14,    /* levels with at most this many free unknowns (default 20000000, i.e. up to
                                256^3; the element operator at most 3000000, i.e. 128^3, where it measured
                                faster) and more than ECMG_OPT_PERSISTENT run the whole
                                tolerance-stopped solve as ONE cooperative launch of TMA z-marching passes
                                (no per-iteration kernel launches); 0: the CUDA-graph loop of K1 / K2 */
  ECMG_OPT_BETA_FLY = 15,    /* element-beta path, cubic cells, analytic beta (C3, C5, layers, beta = 1 with
                                Robin / Neumann faces): 1: the TMA element kernels form beta_e in registers
                                from per-axis tables (the same function the beta array is filled with,
                                bitwise) instead of reading the array, 16 B less HBM traffic per unknown and
                                iteration; 0 (default): read the array (measured as fast: the element
                                kernels are latency bound at 2 CTAs per SM, not HBM bound) */
  ECMG_OPT_SLAB_HYBRID = 16, /* z-slabs: 1 (default) the replicated levels (before the first sharded one)
                                run through the single-GPU path (one-CTA / persistent / CUDA-graph solves,
                                setup ahead) on every rank, then the slab driver takes over; 0: the slab
                                driver's host-driven loop for every level (ablation) */
  ECMG_OPT_UNFUSED = 17,     /* ablation: 1 = fixed-count (eps <= 0) constant-stencil solves run the unfused
                                textbook PCG sequence -- w = A p, p.w, two axpys, z = D^-1 r, r.z, r.r and the
                                p update as separate passes (144 B per unknown and iteration instead of the
                                fused 64 B); 0 (default): the fused K1 / K2 kernels */
  ECMG_OPT_SHARD_MIN = 18,   /* z-slabs: a level is split across the ranks only if its z extent n satisfies
                                n % 4P == 0, n / P >= 16 (ecmg_slab_partition) and n >= this value (default
                                256); smaller levels are solved replicated on every rank. A split level pays
                                two allreduces and two finalize launches per iteration (~35-50 us), more
                                than a whole 128^3 iteration on one GPU (~29 us) */
  ECMG_OPT_XDEFER = 19,      /* 1 (default): the launched constant-stencil TMA K2 writes x every second iteration
                                only (x_{k+2} = x_k + alpha_k p_k + alpha_{k+1} p_{k+1}, the two roundings of two
                                single updates: bitwise the same iterates; 60 instead of 64 B per unknown and
                                iteration); 2: also the launched element-operator K2 (beta from the array,
                                per-face alpha; 76 instead of 80 B -- bitwise too, but measured slower: those
                                kernels are issue bound, C3 256^3 0.256 -> 0.261-0.285 ms, C5 1024^3 16.0-16.5 ->
                                16.5-16.7 ms per iteration; ablation); 0: x updated in every K2 */
  ECMG_OPT_P0_INIT = 22,     /* constant-stencil TMA kernels on one GPU (the launched K1 / K2 and the cooperative
                                one-launch solves): 1 (default) the init pass stores
                                p_0 = D^-1 r_0 instead of r_0; the first K1 reads it (no transform, no store)
                                and the first K2 forms r_0 = D p_0 instead of reading r -- 16 B per unknown
                                less in iteration 0. r_0 carries one extra rounding (<= 1 ulp; exact for plain
                                CG, D = 1), so iterates agree with value 0 to rounding, not bitwise; 0: r_0
                                stored, p_0 formed by the first K1 */
  ECMG_OPT_RICH_FUSED = 21,  /* ecmg_run / ecmg_run_fixed, constant-stencil TMA path on one GPU: 1 (default) the finest
                                level's true-residual pass (which reads x and scatters u_h anyway) also forms
                                u~_h = EXP_true(u_h, u_2h) at its nodes -- the same expression as the EXP_true
                                kernel, bit for bit -- so x is read once instead of u_h being read back (33
                                instead of 41 B per fine node for the two steps); 0: the separate EXP_true
                                kernel (ablation). ecmg_richardson always runs the separate kernel */
  ECMG_OPT_RHS_SYM = 20,     /* C4 (f a function of r only) on a level that is a cube in n, h, lo and free box: the
                                volume load is invariant under permutations of the node indices, so about a
                                third of the 31^3-node tiles is evaluated and the others are written as
                                permuted copies (k_rhs_c4_sym; equal to the plain kernel up to rounding
                                order). Value = the smallest free-box extent that uses it (default 248, i.e.
                                256^3 and larger); 0: never (ablation) */
  ECMG_OPT_SETUP_CTAS = 11,  /* tuning: CTAs per SM of the fp64-ALU-bound volume-load kernel when it runs
                                ahead (0 = one CTA per work item, the full grid) */
  ECMG_OPT_VIRTUAL_SLABS = 6 /* P in 2..16: run the z-slab decomposition with P slabs on this one GPU
                                (device copies stand in for the NCCL halo messages, an in-order sum
                                kernel for the allreduce; the multi-GPU test fixture); 0 or 1: off */
} ecmg_option;
int ecmg_set_option(ecmg_grid* grid, int option, int value);

typedef struct {
  int iterations;        /* JCG iterations performed (number of A.p products); DSOLVE levels: iterations of
                            the 1e-14 JCG surrogate (reading A12) */
  double rel_res_recur;  /* ||r_k||_2 / ||f_h||_2 from the CG recurrence at exit */
  double rel_res_true;   /* "RRe": ||f_h - A_h u_h||_2 / ||f_h||_2 recomputed at exit */
  double norm_b;         /* ||f_h||_2 over free rows (lifted RHS) */
  int converged;
  int status;            /* ecmg_status of this level */
  double ms_setup, ms_exp, ms_solve, ms_rich;  /* device time (CUDA events) of the level's phases: waiting for /
                            running the setup, EXP_finite, the JCG solve incl. its true-residual pass, EXP_true.
                            With ECMG_OPT_RICH_FUSED the finest level's EXP_true is formed inside the solve's
                            last pass: it is then part of ms_solve, and ms_rich is the g_D fill of u~_h only */
} ecmg_stats;

/* JCG solve of level `level` (Alg. 4 l.7-9): textbook PCG with M = diag(A_h),
 * iterate while ||r||_2 > eps ||f_h||_2 (recurrence residual, tested before every iteration
 * including the first; ||f_h|| = 0 -> absolute residual). eps <= 0 runs exactly max_iter
 * iterations (fixed-iteration benchmark / parity mode). max_iter <= 0 -> 10000.
 *   u      device, level-sized: in = initial guess (free nodes; Dirichlet entries ignored),
 *          out = iterate; Dirichlet entries are set to g_D.
 *   stats  may be NULL.
 * Errors: ECMG_ENOTCONV (stats filled, u holds the last iterate), ECMG_EBREAKDOWN, ECMG_EDIAG,
 * ECMG_EINVAL (no problem bound, level out of range). */
int ecmg_solve_level(ecmg_grid* grid, int level, double eps, int max_iter, double* u, ecmg_stats* stats);

/* EXP_finite (Alg. 4 l.6): W_h on level `level` (>= 2) from u_2h (level-1) and
 * u_4h (level-2): corners by Eq. (jiedian) (5U^1-U^0)/4, edge midpoints by Eq. (zhongdian),
 * all other nodes by 20-node Serendipity interpolation of Eq. (inter) (or Remark 2's Lagrange
 * variant, ECMG_OPT_EXP_VARIANT); Dirichlet nodes get g_D. All three device arrays.
 * Requires cells divisible by 4 per axis on `level`. Errors: ECMG_EMISMATCH, ECMG_EINVAL. */
int ecmg_prolongate_extrapolate(ecmg_grid* grid, int level, const double* u2h, const double* u4h, double* w);

/* EXP_true (Alg. 4 l.10): u~_h = (4U^1 - U^0)/3 at 2h nodes (Eq. t1) and the
 * Chen-Lin formula (Eq. chenlin) at 2h edge centres, averaged over the face / space diagonals at
 * face and cell centres; Dirichlet nodes get g_D. uh: level `level`, u2h: level-1, ut: level. */
int ecmg_richardson(ecmg_grid* grid, int level, const double* uh, const double* u2h, double* ut);

/* Alg. 4 end to end: DSOLVE on levels 0 and 1, then for k = 2..num_levels-1:
 * setup(k), W_k = EXP_finite(u_{k-1}, u_{k-2}), JCG(eps) from W_k, u~_k = EXP_true(u_k, u_{k-1}).
 *   per_level  host array [num_levels] or NULL
 *   u_fine     finest-level u_h (device or host pointer; a host pointer is filled by a D2H copy
 *              inside the call)
 *   ut_fine    finest-level u~_h (device or host) or NULL
 * Returns the first failing level's status (ECMG_ENOTCONV etc.) or ECMG_OK. */
int ecmg_run(ecmg_grid* grid, double eps, ecmg_stats* per_level, double* u_fine, double* ut_fine);

/* Alg. 3, the original ECMG the paper starts from: the same cascade, but each ECMG
 * level j = 1..L (L = num_levels - 2) runs exactly m_j = ceil(m_L * ratio^(L-j)) iterations
 * (Eq. ee; the paper's suggested setting is m_L = 4, ratio = 4) instead of the
 * relative-residual test. The paper's Alg. 3 uses plain CG: set ECMG_OPT_PRECOND = 0 for that.
 * Single GPU only (ECMG_EINVAL with slabs). Outputs as ecmg_run. */
int ecmg_run_fixed(ecmg_grid* grid, int m_L, double ratio, ecmg_stats* per_level, double* u_fine, double* ut_fine);

/* Diagnostics used by the parity tests (same kernels as the solve):
 * ecmg_apply_operator: q = A_ff p on free nodes, q = 0 on Dirichlet nodes (p's Dirichlet entries
 *   are ignored). ecmg_level_rhs: lifted right-hand side b_f = F_f + G_f - A_fD g_D on free nodes,
 *   0 on Dirichlet nodes, and ||b_f||_2. Both arrays device, level-sized. */
int ecmg_apply_operator(ecmg_grid* grid, int level, const double* p, double* q);
int ecmg_level_rhs(ecmg_grid* grid, int level, double* b, double* norm_b);

/* Level geometry: cells per axis, number of nodes of the caller-visible vector of this rank, and
 * the half-open z node-plane range [z_lo, z_hi) it holds: the whole level [0, nz+1) on one GPU
 * (and with virtual slabs); on NCCL ranks the rank's slab of a sharded level. */
int ecmg_level_shape(const ecmg_grid* grid, int level, int n_cells3[3], long long* nodes, int* z_lo, int* z_hi);

/* z-slab partition, a pure host function usable without a GPU: a level with
 * n_cells_z cells can be sharded over nranks iff n % (4 nranks) == 0 and n / nranks >= 16; then rank r
 * owns node planes [r n/P, (r+1) n/P) (the last rank also plane n). Returns 1 (sharded, range
 * filled), 0 (replicated: [0, n+1)), or ECMG_EINVAL. A grid additionally keeps levels with
 * n < ECMG_OPT_SHARD_MIN (default 256) replicated; ecmg_level_shape reports the layout it uses. */
int ecmg_slab_partition(int n_cells_z, int nranks, int rank, int* z_lo, int* z_hi);

/* NCCL unique id for ecmg_dist.nccl_id: rank 0 calls this and broadcasts the 128 bytes (e.g. with
 * torch.distributed) before every rank calls ecmg_create_grid. Errors: ECMG_ENCCL. */
int ecmg_nccl_unique_id(unsigned char id[128]);

/* Device time of the last solve's JCG iteration kernels (K1 + K2), for roofline reporting:
 * total milliseconds and number of iterations timed (CUDA events around the iteration loop). */
int ecmg_last_jcg_timing(const ecmg_grid* grid, double* ms, int* iterations, long long* free_unknowns);

/* Number of CUDA kernels libecmg has launched in this process (all grids; monotone counter).
 * bench.py reports the difference across its timed region as "gpu_launches". */
long long ecmg_kernel_launches(void);

int ecmg_destroy_grid(ecmg_grid* grid);
const char* ecmg_strerror(int status);

#ifdef __cplusplus
}
#endif
#endif /* ECMG_H */
