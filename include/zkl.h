/*
 * zkl — B200-native tlookup prover (zkLLM, arXiv 2404.16109, §4 Protocol 1) : the C ABI.
 *
 * The hot path of Protocol 1 without the commitments:
 *   zkl_tlookup_prepare  tlookup-Prep: m_i = |{j : S_j = T_i}|
 *                        (Eq. hab22-coefs)
 *   zkl_tlookup_prove    tlookup-Prove: A = 1/(beta+S), B = 1/(beta+T)
 *                        (Eq. hab22-invs), then the sumcheck
 *                        of Eq. tlookup-sumcheck
 *   zkl_sumcheck_prove   the same sumcheck on caller-supplied A, S, B, T, m
 * plus the boundary encoders (import/export of field vectors) and the table handle.
 *
 * Field: BLS12-381 scalar field Fr, r = 0x73eda753299d7d483339d80809a1d80553bda402fffe5bfeffffffff00000001
 * (PAPER.md:543, 627).
 *
 * Conventions ("readings"):
 *   - a host field element (zkl_fr) is canonical: 8 little-endian 32-bit words, value < r;
 *   - a device field vector (zkl_vec) is Montgomery form (x * 2^256 mod r) in limb-interleaved
 *     SoA layout: limb l of element i at limbs[l*n + i]; limbs must be 16-byte aligned and n a
 *     multiple of 4 (or n < 4);
 *   - coordinate 0 of the hypercube is the MSB of the row-major index; table index j = x mod N;
 *     the table's eq point is u[log2(D/N):];
 *   - sumcheck round k (1-based) binds coordinate d-k (LSB first) with r[k-1]; round polynomial
 *     g_k is returned by its values g_k(0), g_k(1), g_k(2), g_k(3);
 *   - weights (1, alpha1, alpha2) of the three constraints (paper: alpha2 = alpha1^2);
 *     the claimed sum is alpha1 + alpha2 (ZKL_VARIANT_PAPER) or alpha1 (ZKL_VARIANT_LOGUP);
 *   - final evaluations: A(v), S(v), B(v'), T(v'), m(v') with v_c = r[d-1-c], v' = v[d-n:].
 *
 * Ownership: the caller owns every device buffer (inputs, outputs, the workspace and the table
 * memory).  The library owns only the opaque zkl_ctx / zkl_table objects (paired create/destroy).
 * Streams: all device work is enqueued on the ctx's CUDA stream (plus internal events); every call
 * returns when its host-visible outputs are ready and its device outputs are complete.
 * Errors: every int-returning call returns a zkl_status; err_index (when given) is set to the
 * smallest offending index, or -1.  Outputs are unspecified on error.  No exception or abort
 * crosses the ABI.  An asynchronous CUDA fault poisons the ctx (ZKL_E_STATE afterwards).
 * Multi-rank (nranks > 1) calls are collective: every rank passes identical scalars/challenges and
 * its own contiguous slice S_local = S[rank*D/P, (rank+1)*D/P) (top log2 P coordinates = rank).
 */
#ifndef ZKL_H
#define ZKL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { uint32_t w[8]; } zkl_fr;                  /* canonical, little-endian, < r */
typedef struct { uint32_t* limbs; uint64_t n; } zkl_vec;   /* device, SoA Montgomery */
typedef struct zkl_ctx zkl_ctx;
typedef struct zkl_table zkl_table;
typedef struct zkl_group zkl_group;

typedef enum {
    ZKL_OK = 0,
    ZKL_E_ARG = 1,            /* null pointer / bad argument */
    ZKL_E_SHAPE = 2,          /* D, N not powers of two, N > D, P does not divide D, ... */
    ZKL_E_NONCANONICAL = 3,   /* an input element >= r (err_index = element) */
    ZKL_E_DUP_TABLE = 4,      /* T has repeated entries (err_index = smallest later duplicate) */
    ZKL_E_NOT_IN_TABLE = 5,   /* S_i not in T (err_index = smallest global i) */
    ZKL_E_DIV_ZERO_T = 6,     /* beta + T_j = 0 (err_index = smallest j; checked before S) */
    ZKL_E_DIV_ZERO_S = 7,     /* beta + S_i = 0 (err_index = smallest global i) */
    ZKL_E_CUDA = 8,
    ZKL_E_NCCL = 9,
    ZKL_E_OOM = 10,           /* workspace / table memory too small */
    ZKL_E_STATE = 11          /* ctx poisoned by an earlier asynchronous fault */
} zkl_status;

typedef enum { ZKL_VARIANT_PAPER = 0, ZKL_VARIANT_LOGUP = 1 } zkl_variant;

/* Verifier challenges, canonical, host memory.  beta is the paper's beta (the north star's X);
 * u[0..d-1] is the eq point (u[0] pairs with coordinate 0, the MSB); r[k-1] is round k's challenge. */
typedef struct {
    zkl_fr beta, alpha1, alpha2;
    const zkl_fr* u;
    const zkl_fr* r;
} zkl_challenges;

typedef struct { zkl_fr A, S, B, T, m; } zkl_final_evals;

/* ---------------------------------------------------------------- context */
const char* zkl_strerror(int status);
/* Create a context on `device` enqueuing on `cuda_stream` (cudaStream_t; NULL = legacy stream). */
int zkl_ctx_create(int device, void* cuda_stream, zkl_ctx** out);
/* Multi-rank context: nccl_id is the 128-byte ncclUniqueId from rank 0 (zkl_nccl_unique_id),
 * broadcast by the caller (torch.distributed).  NCCL is loaded at run time (libnccl.so.2). */
int zkl_nccl_unique_id(uint8_t id[128]);
int zkl_ctx_create_dist(int device, void* cuda_stream, const uint8_t nccl_id[128], int rank, int nranks,
                        zkl_ctx** out);
/* Loopback communicator: P virtual ranks in ONE process on one device, one host thread per rank, each with
 * its own ctx.  Collectives are host barriers around device copies through the group's staging memory (no
 * kernel waits on another rank's kernel).  For testing the multi-rank path (partition, exchange, replicated
 * rounds) without NCCL; max_N bounds the table size.  The group must outlive its contexts. */
int zkl_group_create(int device, int nranks, uint64_t max_D_local, uint64_t max_N, zkl_group** out);
void zkl_group_destroy(zkl_group* group);
int zkl_ctx_create_loopback(int device, void* cuda_stream, zkl_group* group, int rank, zkl_ctx** out);
void zkl_ctx_destroy(zkl_ctx* ctx);
const char* zkl_last_error(const zkl_ctx* ctx);
/* Workspace for prepare/prove/sumcheck with local length D_local and table size N (bytes, 256-B aligned). */
size_t zkl_workspace_bytes(uint64_t D_local, uint64_t N, int nranks);
int zkl_ctx_set_workspace(zkl_ctx* ctx, void* device_ptr, size_t bytes);
/* Kernel launches issued by this ctx since creation (for launch accounting). */
uint64_t zkl_ctx_launch_count(const zkl_ctx* ctx);
/* Per-launch timing: when on, every launch is bracketed by CUDA events on its stream (<= 256 launches
 * are recorded, then recording stops).  zkl_ctx_profile_read synchronizes, writes up to `cap` kernel names
 * (name_len bytes each, NUL-terminated), durations in ms, (if non-NULL) start times relative to the first
 * recorded launch and the stream of each launch (0 = the ctx stream, 1 = table-side stream, 2 = aux
 * stream, 3 = the low-priority histogram stream of async mode), returns the count, and clears the record. */
int zkl_ctx_set_profiling(zkl_ctx* ctx, int on);
int zkl_ctx_profile_read(zkl_ctx* ctx, char* names, int name_len, float* ms, float* start_ms, int* stream_tag,
                         int cap);

/* ---------------------------------------------------------------- boundary encode (a1) */
/* canonical 32-byte LE elements (host or device, AoS) -> dst (SoA Montgomery).  E_NONCANONICAL(i). */
int zkl_vec_import(zkl_ctx* ctx, const void* canon_le32, int src_on_device, zkl_vec dst, int64_t* err_index);
/* signed 64-bit integers (device) -> Fr (x < 0 maps to r - |x|, reading 15). */
int zkl_vec_import_i64(zkl_ctx* ctx, const int64_t* x_dev, zkl_vec dst);
/* function lookup input: dst_i = x_i + alpha_f * y_i from int32 device arrays. */
int zkl_vec_import_pair(zkl_ctx* ctx, const int32_t* x_dev, const int32_t* y_dev, const zkl_fr* alpha_f,
                        zkl_vec dst);
/* src (SoA Montgomery) -> canonical 32-byte LE elements (host or device, AoS). */
int zkl_vec_export(zkl_ctx* ctx, zkl_vec src, void* canon_le32, int dst_on_device);

/* ---------------------------------------------------------------- matmul sumcheck
 * PAPER.md:463-467 (§5.1.1, Eq. matmul): C = A B with A in F^{m x n}, B in F^{n x p} is proved by the sumcheck
 *     C~(u, v) = sum_{i in {0,1}^{log2 n}} A~(u, i) B~(i, v).
 * A, B: quantised int32 entries (mapped into F as x mod r), row-major, DEVICE, m x n and n x p;
 * m, n, p powers of two, n <= 2^39.  u (log2 m), v (log2 p), r (log2 n): canonical challenges, HOST (u[0] pairs
 * with the row MSB; r[k-1] is round k's challenge, binding coordinate log2(n) - k of i, pairs (2y, 2y+1)).
 * Outputs: a_i = A~(u, i) and b_i = B~(i, v) into a_out / b_out (device SoA Montgomery vectors of n; limbs may be
 * NULL), claim = sum_i a_i b_i = C~(u, v) (host), round_evals[k-1][t] = g_k(t), t = 0, 1, 2 (host, 3 log2 n
 * values), finals = [a~(w), b~(w)] at the bound point (host).  Uses the ctx workspace (zkl_matmul_workspace_bytes;
 * it replaces any prepared index keys).  Synchronous only (E_STATE in async mode).  E_SHAPE, E_NONCANONICAL, E_OOM. */
size_t zkl_matmul_workspace_bytes(uint64_t m, uint64_t n, uint64_t p);
int zkl_matmul_prove(zkl_ctx* ctx, const int32_t* A, const int32_t* B, uint64_t m, uint64_t n, uint64_t p,
                     const zkl_fr* u, const zkl_fr* v, const zkl_fr* r, zkl_vec a_out, zkl_vec b_out, zkl_fr* claim,
                     zkl_fr* round_evals, zkl_fr* finals);

/* ---------------------------------------------------------------- Hyrax / Pedersen commitments
 * PAPER.md:187-203 (§3.4; Hyrax = Pedersen without trusted setup, homomorphic), Protocol 1 lines 261, 267-269, 275.
 * Group: BLS12-381 G1 (y^2 = x^3 + 4 over F_q).  A vector S of D = rows x cols Fr elements (row-major) commits to
 * rows points C_j = sum_i S[j cols + i] G_i + rho_j H.  G_0..G_{cols-1}, H are public: hashed to the curve from
 * labels by try-and-increment, so no trusted setup.  Points leave the library affine with
 * canonical little-endian F_q coordinates (infinity = 1 for the point at infinity, coordinates 0). */
typedef struct {
    uint32_t x[12];
    uint32_t y[12];
    uint32_t infinity;
} zkl_g1;

/* Device bytes of the public parameters for `cols` generators (+ H), with their 4-bit window tables. */
size_t zkl_hyrax_pp_bytes(uint64_t cols);
/* Derive the generators and tables into caller-owned device memory pp (>= zkl_hyrax_pp_bytes). cols power of 2. */
int zkl_hyrax_setup(zkl_ctx* ctx, uint64_t cols, void* pp_dev, size_t pp_bytes);
/* Copy G_0..G_{cols-1}, H (cols + 1 points) to host memory. */
int zkl_hyrax_export_generators(zkl_ctx* ctx, const void* pp_dev, uint64_t cols, zkl_g1* out_host);
/* Workspace bytes (ctx workspace) of zkl_hyrax_commit / zkl_hyrax_prove_eval for D elements in rows of cols. */
size_t zkl_hyrax_workspace_bytes(uint64_t D, uint64_t cols);
/* Commit(S, rho; pp): C_host[j] for j < D / cols.  rho: host, D / cols canonical blinds, or NULL (no hiding, as
 * tlookup-Setup's Commit(T; 0)).  S: device SoA Montgomery vector (n >= D).  E_SHAPE, E_NONCANONICAL,
 * E_OOM. */
int zkl_hyrax_commit(zkl_ctx* ctx, const void* pp_dev, uint64_t cols, zkl_vec S, uint64_t D, const zkl_fr* rho,
                     zkl_g1* C_host);
/* ProveEval in the row-restriction form: v = (v_rows, v_cols), host, log2 D canonical values, the
 * first log2(D / cols) for the row index (high bits).  w_out (device, cols) = sum_j e~(v_rows, j) S_row_j, and
 * y_host = <w, e~(v_cols, .)> = S~(v).  The verifier checks Com(w, sum_j e~ rho_j) = sum_j e~(v_rows, j) C_j; the
 * O(log D) inner-product argument on w is not part of this build. */
int zkl_hyrax_prove_eval(zkl_ctx* ctx, zkl_vec S, uint64_t D, uint64_t cols, const zkl_fr* v, zkl_vec w_out,
                         zkl_fr* y_host);

/* ---------------------------------------------------------------- Protocol 1 with its commitments (§8(f1) + (f3))
 * PAPER.md:252-278 (Protocol 1, tlookup) in the function-lookup form of PAPER.md:287 (X + alpha_f Y in
 * T_X + alpha_f T_Y), non-interactive: every message is absorbed into a SHA-256 transcript before the challenge
 * that follows it:
 *   h = SHA256("zkl-p1-v1" || seed || le64(D) || le64(N) || le32(variant) || le64(cols));
 *   absorb [T_X], [T_Y] (tlookup-Setup, Commit(T; 0)), [X], [Y]  -> alpha_f;  S = X + alpha_f Y, [S] = [X] + alpha_f [Y];
 *   m (tlookup-Prep), absorb [m]  -> beta;  A, B, absorb [A], [B]  -> alpha1 (alpha2 = alpha1^2), u;
 *   the sumcheck with r_k from the transcript (as zkl_tlookup_prove_fs);
 *   row-restriction proofs of evaluation (zkl_hyrax_prove_eval) of A, X, Y at v and of T_X, T_Y, m, B at v'.
 * Commitments are Hyrax rows of `cols` entries (cols | N | D), with no hiding (blinds 0) in this build.
 * x, y (D int32) and tx, ty (N int32, tx a contiguous range) are device arrays; pp from zkl_hyrax_setup(cols).
 * Every output pointer is HOST memory the caller provides: C_X, C_Y, C_A (D / cols points), C_TX, C_TY, C_m, C_B
 * (N / cols points), round_evals (log2 D x 4), derived (3 + 2 log2 D: beta, alpha1, alpha2, u, r), the w vectors
 * (cols canonical values each) and the y values.  Single rank, synchronous.  The context's workspace must hold
 * zkl_workspace_bytes(D, N, 1); the Hyrax steps use a buffer the context owns. */
typedef struct {
    zkl_g1 *C_X, *C_Y, *C_TX, *C_TY, *C_m, *C_A, *C_B;
    zkl_fr* round_evals;
    zkl_final_evals finals;
    zkl_fr alpha_f;
    zkl_fr* derived;
    zkl_fr *w_A, *w_X, *w_Y, *w_TX, *w_TY, *w_m, *w_B;
    zkl_fr y_A, y_X, y_Y, y_TX, y_TY, y_m, y_B;
} zkl_p1_proof;

int zkl_tlookup_prove_p1(zkl_ctx* ctx, const void* pp_dev, uint64_t cols, const int32_t* x_dev, const int32_t* y_dev,
                         uint64_t D, const int32_t* tx_dev, const int32_t* ty_dev, uint64_t N, const uint8_t seed[32],
                         zkl_variant variant, zkl_p1_proof* out);

/* ---------------------------------------------------------------- async mode (many instances)
 * With async on, zkl_tlookup_prepare(_pair), zkl_tlookup_prove(_fs) and zkl_sumcheck_prove validate their
 * arguments, enqueue their kernels on the ctx stream and return ZKL_OK at once; their outputs (m is on the device
 * as usual; round_evals, finals, derived and err_index in HOST memory, which must stay valid) are delivered by
 * zkl_ctx_wait, which also returns the first error of the pending calls, in call order (later calls' outputs
 * are then not delivered).  At most one pending prepare and one pending prove per ctx (else E_STATE): K
 * instances in flight = K contexts, each with its own CUDA stream and workspace, so the GPU overlaps one
 * instance's latency-bound tail with another's bandwidth/ALU-bound rounds.  At P > 1 (NCCL) the prepare's histogram
 * and its all-reduce run on the low-priority stream and the proof's collectives are ordered after them; with the
 * loopback communicator (host-synchronising collectives) the prepare stays synchronous.
 * A proof whose prepared keys missed falls back to the inversion path synchronously inside zkl_ctx_wait. */
int zkl_ctx_set_async(zkl_ctx* ctx, int on);
int zkl_ctx_wait(zkl_ctx* ctx);

/* ---------------------------------------------------------------- table handle (a2) */
/* Device memory the caller provides for a table of N entries. */
size_t zkl_table_bytes(uint64_t N);
/* Validate (N power of two, entries distinct) and index T (a copy is kept in `mem`).
 * E_SHAPE, E_DUP_TABLE(smallest later duplicate), E_OOM. */
int zkl_table_create(zkl_ctx* ctx, zkl_vec T, void* mem, size_t mem_bytes, zkl_table** out, int64_t* err_index);
void zkl_table_destroy(zkl_table* table);
/* Function-lookup fast path (a3): declare that T_j = tx_j + alpha_f ty_j with tx the contiguous range
 * tx_0 + j (int32 device arrays of N entries; checked on the device, ty copied into the table memory).  Then
 * zkl_tlookup_prepare_pair with the same alpha_f indexes (x, y) as j = x - tx_0 (checked: ty_j == y) instead of
 * hashing; any pair failing the check sends the prepare through the exact hash index.  E_ARG if T is not of that
 * form (the table stays usable without the fast path). */
int zkl_table_attach_pair(zkl_ctx* ctx, zkl_table* table, const int32_t* tx_dev, const int32_t* ty_dev,
                          const zkl_fr* alpha_f);

/* ---------------------------------------------------------------- the hot path */
/* tlookup-Prep (Eq. hab22-coefs): m_dev[j] = #{i : S_i = T_j}
 * over ALL ranks (u32, device, N entries).  D is the global length.  E_NOT_IN_TABLE(smallest i). */
int zkl_tlookup_prepare(zkl_ctx* ctx, zkl_vec S_local, uint64_t D, const zkl_table* T, uint32_t* m_dev,
                        int64_t* err_index);

/* Function-lookup form of tlookup-Prep (a1 + a3 fused): S_local_out[i] =
 * x_i + alpha_f y_i (int32 device arrays of length D/P; same encoding as zkl_vec_import_pair) is written and
 * counted into m_dev in one pass over x, y.  Same errors as zkl_tlookup_prepare.
 * S_local_out.limbs == NULL: S stays VIRTUAL -- only the table index of every lookup is kept (in the workspace);
 * the following zkl_tlookup_prove / _prove_fs on this context, table and D takes S_local.limbs == NULL and reads
 * S_i = T_key(i) (and A_i = B_key(i)) from the table instead of a D-sized vector (S is committed homomorphically
 * as [X] + alpha [Y], so it need not exist in HBM). */
int zkl_tlookup_prepare_pair(zkl_ctx* ctx, const int32_t* x_dev, const int32_t* y_dev, const zkl_fr* alpha_f,
                             uint64_t D, const zkl_table* T, zkl_vec S_local_out, uint32_t* m_dev,
                             int64_t* err_index);

/* tlookup-Prove: A_local_out = 1/(beta + S_local), B_out = 1/(beta + T)
 * (LOGUP: m/(beta + T)), then the log2(D)-round sumcheck of Eq. tlookup-sumcheck.
 * round_evals: host, log2(D) x 4 canonical values g_k(0..3), k = 1..log2 D.  finals: host.
 * A_local_out / B_out may have limbs == NULL (not materialised for the caller; A is still computed).
 * E_DIV_ZERO_T / E_DIV_ZERO_S (err_index), E_SHAPE. */
int zkl_tlookup_prove(zkl_ctx* ctx, zkl_vec S_local, uint64_t D, const zkl_table* T, const uint32_t* m_dev,
                      const zkl_challenges* ch, zkl_variant variant, zkl_vec A_local_out, zkl_vec B_out,
                      zkl_fr* round_evals, zkl_final_evals* finals, int64_t* err_index);

/* The whole step from HOST buffers (the end-to-end call of a function lookup): x, y (D/P int32) and
 * tx, ty (N int32, tx a contiguous range; T_j = tx_j + alpha_f ty_j) are copied to device buffers the context
 * owns (allocated on first use, freed by zkl_ctx_destroy), then T is imported and indexed (zkl_table_create +
 * zkl_table_attach_pair), prepare_pair runs with a virtual S, and zkl_tlookup_prove writes round_evals and
 * finals (host) -- exactly the device-resident step, with the host->device copies inside the call.  Pinned host
 * memory makes the copies run at the PCIe rate.  m_out (host, N u32) may be NULL.  Errors as the calls it makes;
 * E_ARG if tx is not a range (use the device-buffer calls with the hash index then).  Synchronous. */
int zkl_tlookup_prove_pair_host(zkl_ctx* ctx, const int32_t* x_host, const int32_t* y_host, uint64_t D,
                                const int32_t* tx_host, const int32_t* ty_host, uint64_t N, const zkl_fr* alpha_f,
                                const zkl_challenges* ch, zkl_variant variant, zkl_fr* round_evals,
                                zkl_final_evals* finals, uint32_t* m_out, int64_t* err_index);

/* Fiat-Shamir (non-interactive) tlookup-Prove: the same proof, with beta, alpha1, alpha2 = alpha1^2, u and every
 * r_k derived on the device from a SHA-256 transcript: h_0 = SHA256("zkl-fs-v1" || seed ||
 * le64(D) || le64(N) || le32(variant)); chal(label, i) = SHA256(h || label || le32(i)) mod r; beta = chal("beta",0),
 * alpha1 = chal("alpha",0), u_c = chal("u",c); after round k, h_k = SHA256(h_{k-1} || "g" || le32(k) ||
 * g_k(0..3) as 32-byte LE) and r_k = chal("r", k).  `seed` (32 bytes) stands for the commitments sent before
 * beta ([T], [S], [m]; commitments are outside this path).  derived (host, 3 + 2 log2 D): beta, alpha1,
 * alpha2, u[0..d-1], r[0..d-1], canonical.  Single rank; D >= 2. */
int zkl_tlookup_prove_fs(zkl_ctx* ctx, zkl_vec S_local, uint64_t D, const zkl_table* T, const uint32_t* m_dev,
                         const uint8_t seed[32], zkl_variant variant, zkl_vec A_local_out, zkl_vec B_out,
                         zkl_fr* round_evals, zkl_final_evals* finals, zkl_fr* derived, int64_t* err_index);

/* The sumcheck alone on caller-supplied vectors (any values: tamper trials, benchmarking); inputs are
 * never modified.  m_fr is m as field elements (SoA Montgomery, N).  B is the variant's B. */
int zkl_sumcheck_prove(zkl_ctx* ctx, zkl_vec A_local, zkl_vec S_local, uint64_t D, zkl_vec B, zkl_vec T,
                       zkl_vec m_fr, const zkl_challenges* ch, zkl_variant variant, zkl_fr* round_evals,
                       zkl_final_evals* finals);

#ifdef __cplusplus
}
#endif
#endif /* ZKL_H */
