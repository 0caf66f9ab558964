// irk-b200 internal definitions (not part of the C-ABI).
//
// Device block layout ("column-pair interleaved"): an nb x nb fp64 block is
// stored as P = ceil(nb/2) column pairs; pair p holds rows 0..nb-1, each row
// contributing the 16-byte vector (B[a][2p], B[a][2p+1]).  Element (a, b)
// lives at double offset ((b>>1)*nb + a)*2 + (b&1).  A warp whose lanes walk
// consecutive rows a of one pair therefore issues perfectly coalesced 128-bit
// loads, and a thread that owns row a multiplies both columns of the pair
// with a broadcast x[2p..2p+1].  Odd nb pads the last pair's second column
// with zeros (block size nb * 2P doubles).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/irkb200.h"

namespace irk {

void set_error(const std::string& msg);
int fail_cuda(cudaError_t e, const char* what, const char* file, int line);

#define IRK_CK(call)                                                          \
    do {                                                                      \
        cudaError_t _e = (call);                                              \
        if (_e != cudaSuccess) return ::irk::fail_cuda(_e, #call, __FILE__, __LINE__); \
    } while (0)

void count_launch();
// after every kernel launch: count it (irk_launch_count) and check the launch
#define IRK_LAUNCHED()                                                        \
    do {                                                                      \
        ::irk::count_launch();                                                \
        IRK_CK(cudaGetLastError());                                           \
    } while (0)

#define IRK_ARG(cond, msg)                                                    \
    do {                                                                      \
        if (!(cond)) { ::irk::set_error(std::string("invalid argument: ") + (msg)); return IRK_EINVAL; } \
    } while (0)

#define IRK_TRY(expr)                                                         \
    do { int _rc = (expr); if (_rc != IRK_OK) return _rc; } while (0)

// ---- programmatic dependent launch (PDL) -----------------------------------
// Hot kernels are launched with programmatic stream serialisation: each one
// triggers its dependents at entry (every CTA of a single-wave grid is then
// resident, so a waiting dependent can never block it), and waits for its
// predecessor (griddepcontrol.wait) after its prologue, before its first
// global read or write.  The next kernel's CTAs launch and initialise their
// shared-memory pipelines (mbarriers, rings) during the previous kernel's
// drain.  IRK_PDL=0 disables it (plain stream order).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_if(bool on, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                 cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = (on && pdl_enabled()) ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Pivot blocks formed inside the inverse kernel (factor level 0, no Schur update):
// D_{j,k} = keep[diag_j] ? fl(alpha J_jj) + fl(coef_k M_j) : 0 (build_stage_matrix,
// precond.py:48-54, the rounding of the Schur phase's initialisation).
struct InvForm {
    const double* J = nullptr;      // stage-shared Jacobian blocks (pattern order)
    const int32_t* diag = nullptr;  // diagonal block position per element
    const uint8_t* keep = nullptr;
    const double* M = nullptr;      // mass blocks or NULL
    double* Dst = nullptr;          // pivot blocks (written when store or for pivoted fallback)
    double alpha = 0.0;
    double coef[IRK_MAX_STAGES] = {};
    int store = 0;                  // also write D (export / literal need it)
};

inline int npairs(int nb) { return (nb + 1) / 2; }
inline int64_t block_doubles(int nb) { return (int64_t)nb * 2 * npairs(nb); }

}  // namespace irk

// ---------------------------------------------------------------------------
// opaque handle definitions
// ---------------------------------------------------------------------------
struct irk_ctx {
    int device = 0;
    int num_sms = 148;
    size_t smem_optin = 0;
    size_t smem_per_sm = 0;
};

struct irk_pattern {
    irk_ctx* ctx = nullptr;
    int64_t T = 0, nnzb = 0;
    // host copies (int64, reference layout)
    std::vector<int64_t> h_indptr, h_indices, h_diag;
    // device (int32)
    int32_t* d_indptr = nullptr;   // T+1
    int32_t* d_indices = nullptr;  // nnzb
    int32_t* d_diag = nullptr;     // T
    int32_t* d_rowof = nullptr;    // nnzb: row of each block
    // lower / upper slot maps (lower slot = position among strictly-lower blocks)
    int64_t nlow = 0, nup = 0;
    std::vector<int64_t> h_lptr, h_uptr;  // T+1 each
    int32_t* d_lptr = nullptr;     // T+1
    int32_t* d_uptr = nullptr;     // T+1
    int32_t* d_tpos = nullptr;     // nnzb: position of the transposed block (j,i) for (i,j), -1 if absent
};

struct irk_blocks {
    irk_ctx* ctx = nullptr;
    int nb = 0;
    int64_t count = 0;
    double* d = nullptr;            // count * block_doubles(nb)
};

struct irk_stage_op {
    irk_ctx* ctx = nullptr;
    const irk_pattern* pat = nullptr;
    int s = 0, nb = 0;
    const irk_blocks* J[IRK_MAX_STAGES] = {};
    int64_t jfirst[IRK_MAX_STAGES] = {};   // first block of stage k inside J[k]
    bool shared_j = true;
    const irk_blocks* M = nullptr;
    double alpha = 0.0;                    // multiplies J (=-dt)
    double C[IRK_MAX_STAGES * IRK_MAX_STAGES] = {};  // mass mixing (a_inv)
    // optional halo (distributed): columns >= T_local index the ghost buffer
    int64_t T_local = 0;
    const double* ghost = nullptr;
    int64_t n_ghost = 0;
};

// schedule of one sweep direction: element order grouped by level
struct irk_sched {
    int64_t nlevels = 0;
    std::vector<int64_t> h_lvl_ptr;   // nlevels+1
    int32_t* d_order = nullptr;       // T elements in level order
    std::vector<char> h_trivial;      // level has no kept off-diagonal dependency (fwd: z = y)
};

struct irk_factor {
    irk_ctx* ctx = nullptr;
    const irk_pattern* pat = nullptr;
    int kind = 0;          // IRK_FACTOR_UNCOUPLED | IRK_FACTOR_COUPLED
    int s = 0, nb = 0;
    int simplified = 1;
    int literal = 0;
    uint8_t* d_keep = nullptr;        // nnzb
    // lower factors L[lq][k], diag inverses Dinv[i][k], optional stored diag D[i][k]
    double* d_L = nullptr;
    double* d_Dinv = nullptr;
    double* d_D = nullptr;
    // implicit L (uncoupled, stage-shared J, symmetric keep): L_ij = alpha J_ij Dinv_j is
    // never stored; the forward sweep uses w_j = Dinv_j z_j (d_W, s x T x nb) instead
    bool l_implicit = false;
    bool cpl_pipe = false;            // coupled: element-task pipelined sweeps (element schedules)
    double* d_W = nullptr;
    mutable double* d_Z = nullptr;    // deep sentinel sweeps: z_i of the forward sweep (s x T x nb), lazily allocated
    mutable double* d_Wrhs = nullptr; // multi-RHS apply of a single factor: nrhs x T x nb
    mutable int wrhs = 0;
    uint8_t* d_hasup = nullptr;       // T: row has a kept upper block
    // upper blocks: either implicit (ubase[k] block array at pattern position q,
    // scaled by uscale) or stored U[uq][k] (uscale = 1)
    bool u_stored = false;
    double* d_U = nullptr;
    const double* ubase[IRK_MAX_STAGES] = {};
    double uscale = 1.0;
    bool u_shared = false;            // all stages read the same upper blocks
    // coupled: lower couplings G[i][pair(l,k)] for l>k ; upper couplings either
    // implicit C_kl * M_i or stored Cup[i][pair(k,l)] for k<l
    double* d_G = nullptr;
    double* d_Cup = nullptr;          // stored upper couplings (explicit mode)
    const double* mass = nullptr;     // implicit upper couplings
    double cup_scale[IRK_MAX_STAGES * IRK_MAX_STAGES] = {};
    irk_sched fwd, bwd;
    // persistent-sweep synchronisation: per-task flags (fwd, bwd) + tickets
    unsigned* d_flags = nullptr;
    int* d_ticket = nullptr;
    mutable unsigned epoch = 0;
    int maxdeg = 0;                   // max lower/upper neighbours of a row
    // numeric factorisation state (re-run by irk_factor_refactor)
    void* fargs = nullptr;            // FactorArgs (factor.cu)
    irk_sched fsched;                 // factor tasks by level
    unsigned long long* d_fail = nullptr;
    int* d_fb = nullptr;              // tensor-core inverse: blocks handed to the pivoted kernels
    mutable int fb_optimistic = 0;    // deep schedules: levels run without the per-level fallback launch (factor_numeric)
    bool store_d = false;             // pivot blocks must be kept (store_diag / literal)
    mutable bool d0_unstored = false; // level-0 pivot blocks were formed in the inverse, not stored
    // Schur path: per factor level, its elements and element-major (stage fastest) task codes
    int32_t* d_fs_elems = nullptr;
    int32_t* d_fs_tasks = nullptr;
    std::vector<int64_t> h_fs_eptr;   // nlevels+1 element offsets
    // side stream + events: the inverse of Schur chunk c overlaps the Schur phase of chunk c+1
    mutable cudaStream_t st2 = nullptr;
    mutable std::vector<cudaEvent_t> ev;
    // deep factor schedules (one Schur + inverse launch pair per level, hundreds of levels): the
    // level loop is captured once into a CUDA graph and replayed while the kernel arguments stay
    // the same (factor.cu factor_numeric)
    void* fgraph = nullptr;
    size_t fsmem = 0;
    int maxt = 1;
    const double* cpl_src = nullptr;  // explicit couplings (s*s*T blocks)
    // fused Arnoldi product with an element-partitioned operator (apply.cu halo_pair_ok):
    // the checked (operator, numeric version) pair and its verdict
    unsigned numeric_epoch = 0;       // bumped by every re-factorisation
    mutable const irk_stage_op* halo_op = nullptr;
    mutable unsigned halo_epoch = 0;
    mutable bool halo_ok = false;
    // owned copies when created from explicit host data
    std::vector<irk_blocks*> owned;
};
