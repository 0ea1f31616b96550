/* hfb.h — C ABI of the B200-native timestep engine for Hybrid-Fortran grid programs.
 *
 * This is the drop-in boundary for the reference's data-parallel hot path: running
 * a Hybrid-Fortran program's timestep (its @parallelRegion kernels) over module
 * state arrays. It replaces, one for one:
 *
 *   reference                                              here
 *   ----------------------------------------------------   ------------------------------
 *   hft::interp::MachineState (interp.hpp:49-60)           hfb_ctx (+ hfb_set_scalar_*,
 *     module scalars / ObjectSlot host buffers               hfb_bind_array)
 *   hft::interp::Program (interp.hpp:78-109)               hfb_load_program (built-in apps)
 *   run_gpu_simulated / run_program (interp.hpp:113-122,   hfb_run
 *     interp.cpp:1563-1590) + LaunchStats (:72-76)
 *   hfrt_device_allocate / hfrt_copy_to_device /           hfrt_device_allocate / ...
 *     hfrt_copy_from_device (codegen.cpp:580-600,            (same residency state machine
 *     semantics interp.cpp:1369-1415)                        and errors)
 *   generated kernels hfk<i>_<routine> launched            hfk0_diffuse_step, ... (same
 *     <<<ceil(ext/B), B>>> (codegen.cpp:397-519,             argument order: value scalars
 *     captures :768-843)                                     alphabetical, then arrays)
 *   hft::Error{ErrKind} (diagnostics.hpp:21-52)            hfb_status = 10 + ErrKind
 *
 * Conventions: plain C types only; strings are module/object names (case-insensitive,
 * as MachineState keys are lower-cased). Host buffers stay owned by the caller; device
 * buffers are owned by the context and freed by hfb_destroy. There is no CPU fallback:
 * an unknown app/entry/kernel is HFB_CONFIG, a missing CUDA device is HFB_CUDA.
 * A context is single-threaded (as MachineState is).
 */
#ifndef HFB_H
#define HFB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --- status codes: 10 + hft::ErrKind (diagnostics.hpp:21-32) ------------------- */
typedef int hfb_status;
#define HFB_OK 0
#define HFB_CONFIG 10
#define HFB_RUNTIME 15
#define HFB_RESIDENCY 16
#define HFB_RACE 17
#define HFB_VALIDATION 18
#define HFB_IO 19
#define HFB_CUDA 30 /* CUDA/NCCL error; the generated code's `stop 1` (codegen.cpp:412-418) */

/* message of the last failing call on this thread (never NULL) */
const char* hfb_last_error(void);
/* ABI version of this library */
int hfb_abi_version(void);

/* --- context = MachineState + device residency, bound to one CUDA device ---------- */
typedef struct hfb_ctx hfb_ctx;
hfb_status hfb_create(int device, hfb_ctx** out);
void hfb_destroy(hfb_ctx* ctx);

/* Program: one of the built-in Hybrid-Fortran apps ("diffusion", "damping", "bounded",
 * "surface_flux", "reduction", "dycore"). Creates the app's modules with their scalars
 * (module parameters such as sf_state.ntlm pre-set, interp.cpp:1498-1518). */
hfb_status hfb_load_program(hfb_ctx* ctx, const char* app);

/* Programs can also be generated from Hybrid-Fortran sources (paper_1710_08616_b200/hfc,
 * include/hfb_plugin.h): hfb_load_program(ctx, "<path>.so") loads such a program. */
/* name and state module of the loaded program (NULL before hfb_load_program) */
const char* hfb_program_name(hfb_ctx* ctx);
const char* hfb_program_module(hfb_ctx* ctx);

/* module scalars (MachineState::scalars; interp.hpp:40-47) */
hfb_status hfb_set_scalar_i64(hfb_ctx* ctx, const char* module, const char* name, int64_t v);
hfb_status hfb_set_scalar_f64(hfb_ctx* ctx, const char* module, const char* name, double v);
hfb_status hfb_get_scalar_i64(hfb_ctx* ctx, const char* module, const char* name, int64_t* v);
hfb_status hfb_get_scalar_f64(hfb_ctx* ctx, const char* module, const char* name, double* v);

/* Module array host buffer (ObjectSlot::host; interp.hpp:16-38). `lower`/`upper` are
 * the inclusive declared bounds per dim (rank <= 4, must match the declaration as
 * elaborated from the module scalars). `strides` (elements, per dim) may be NULL for
 * the reference's ArrayValue order (row-major, last subscript fastest,
 * interp.cpp:485-494); Fortran order is strides {1, n1, n1*n2, ...}. The buffer must be
 * dense in some dim permutation. flags: HFB_BIND_PIN page-locks it (cudaHostRegister)
 * so transfers run at full link speed. */
#define HFB_BIND_PIN 1u
hfb_status hfb_bind_array(hfb_ctx* ctx, const char* module, const char* name, int rank,
                          const int64_t* lower, const int64_t* upper, double* host,
                          const int64_t* strides, unsigned flags);

/* Element init flags of a bound array (ArrayValue::init, interp.hpp:16-28; SURVEY §8(b)
 * `init_or_null`): one byte per element at the same element offsets (strides) as the
 * host buffer, caller-owned like the data, NULL unbinds. When flags are bound (or the
 * context runs checked, hfb_set_option "checked"), the device copy carries init flags:
 * hfrt_copy_to_device uploads them, hfrt_device_allocate clears them, kernels set them
 * for the elements they write, a read of an unset element fails with HFB_RUNTIME "read
 * of unset element of '<name>'" (interp.cpp:505-507), and hfrt_copy_from_device writes
 * them back. Arrays bound without flags count as fully set. */
hfb_status hfb_bind_init(hfb_ctx* ctx, const char* module, const char* name, uint8_t* init);

/* --- transfers: the generated-code runtime (codegen.cpp:580-600) ------------------ */
/* residency of a bound array: 0 = Host, 1 = Device, 2 = Both (interp.hpp:30);
 * has_device reports whether a device copy exists */
hfb_status hfb_residency(hfb_ctx* ctx, const char* module, const char* name, int* residency,
                         int* has_device);
hfb_status hfrt_device_allocate(hfb_ctx* ctx, const char* module, const char* name);
hfb_status hfrt_copy_to_device(hfb_ctx* ctx, const char* module, const char* name);
hfb_status hfrt_copy_from_device(hfb_ctx* ctx, const char* module, const char* name);
/* the caller wrote the host buffer after a transfer (write_element's host-side
 * residency flip, interp.cpp:533-538) */
hfb_status hfb_mark_host_modified(hfb_ctx* ctx, const char* module, const char* name);

/* --- entry points: run_gpu_simulated(program, state, entry) ----------------------- */
typedef struct {
  int64_t launches;      /* as the reference's simulated launches count them */
  int64_t threads;       /* (interp.cpp:1417-1475): the generated-code contract */
  int64_t guard_returns;
  int64_t native_launches; /* sm_100a kernels this engine actually launched */
} hfb_launch_stats;

/* Entries are the app's routine names with or without the generated `hfd_` prefix
 * (e.g. "main", "hfd_main", "simulation_run", "diffuse_step", "dycore_step"). The dycore
 * program's per-step entries: "dycore_step", "full_step" (+ column physics), "rk3_step"
 * and "asuca_step" (the ASUCA time scheme, apps/dycore/asuca.h90); the fused kernels take
 * columns of up to 129 levels. Runs to completion on the context's stream and
 * synchronises before returning. */
hfb_status hfb_run(hfb_ctx* ctx, const char* entry, hfb_launch_stats* stats);
/* Same, asynchronously on the context's stream (no host synchronisation); only for
 * entries without transfers. */
hfb_status hfb_enqueue(hfb_ctx* ctx, const char* entry, hfb_launch_stats* stats);
hfb_status hfb_synchronize(hfb_ctx* ctx);
/* the context's CUDA stream (cudaStream_t), for callers that time with events */
void* hfb_stream(hfb_ctx* ctx);
/* Capture `steps` calls of a stream-only entry into a CUDA graph and replay it
 * (launch-overhead-free timestep loop; replaces the generated host driver's per-step
 * launches, codegen.cpp:621-670). Graphs are cached per entry, step count and starting
 * buffer sides. Decomposed contexts on the peer transport are captured too: the halo
 * epochs live in device memory, so every replay signals and waits on fresh epochs
 * (every rank must replay the same sequence). hfb_run_graph synchronises;
 * hfb_enqueue_graph only launches on the context stream. */
hfb_status hfb_run_graph(hfb_ctx* ctx, const char* entry, int64_t steps,
                         hfb_launch_stats* stats);
hfb_status hfb_enqueue_graph(hfb_ctx* ctx, const char* entry, int64_t steps,
                             hfb_launch_stats* stats);

/* --- generated-kernel ABI (codegen.cpp:397-519) ------------------------------------ */
typedef struct {
  uint32_t x, y, z;
} hfb_dim3;

/* Device view of a module array, obtained from a context after a transfer. Opaque
 * layout fields; pass by value to the hfk* entries. */
typedef struct {
  double* origin;       /* element at the lower bounds */
  int64_t pitch;        /* elements between consecutive i rows (j stride) */
  int64_t plane;        /* elements between consecutive k planes */
  int64_t volume;       /* elements between consecutive trailing-dim slices */
  int64_t lower[4], upper[4];
  int32_t rank;
  int32_t roles;        /* packed dim roles (internal) */
  void* slot;           /* owning slot (residency bookkeeping) */
} hfb_array;
hfb_status hfb_device_array(hfb_ctx* ctx, const char* module, const char* name, hfb_array* out);

/* Each hfk* runs exactly the thread set the reference's launch would: threads
 * (blockidx-1)*blockdim+threadidx (+start-1) per axis, guard `it > end` returns
 * (codegen.cpp:495-512). Argument order is the generated one: value scalars
 * alphabetical, then arrays alphabetical (codegen.cpp:436-441). Asynchronous on
 * `stream` (a cudaStream_t, NULL = the context stream of the arrays). */
hfb_status hfk0_diffuse_step(hfb_dim3 grid, hfb_dim3 block, double coef, int32_t k, int32_t nx,
                             int32_t ny, int32_t nz, hfb_array t_new, hfb_array t_old,
                             void* stream);
hfb_status hfk1_diffuse_step(hfb_dim3 grid, hfb_dim3 block, int32_t k, int32_t nx, int32_t ny,
                             int32_t nz, hfb_array t_new, hfb_array t_old, void* stream);
hfb_status hfk0_lateral_and_upper_damping(hfb_dim3 grid, hfb_dim3 block, int32_t k,
                                          double mtratio_bnd, int32_t nx_mn, int32_t nx_mx,
                                          int32_t ny_mn, int32_t ny_mx, int32_t nz_mn,
                                          int32_t nz_mx, double tratio_bnd,
                                          hfb_array dens_ptb_bnd, hfb_array dens_ptb_damp,
                                          hfb_array dens_ref_f, void* stream);
hfb_status hfk0_interior_update(hfb_dim3 grid, hfb_dim3 block, int32_t nx, int32_t ny,
                                hfb_array a, hfb_array b, void* stream);
hfb_status hfk0_sf_slab_flx_tile_run(hfb_dim3 grid, hfb_dim3 block, int32_t nx, int32_t ny,
                                     int32_t tile_land, hfb_array cover_frac,
                                     hfb_array flx_sum_x, hfb_array flx_sum_y,
                                     hfb_array swind, void* stream);

/* --- 2-D horizontal decomposition (new; the reference has none) ------ */
typedef struct {
  int64_t global_nx, global_ny, nz;
  int32_t px, py;      /* process grid */
  int32_t rank;        /* row-major: rank = ry * px + rx */
  int32_t halo;        /* halo width (stencil radius) */
  /* derived by hfb_decomp_init: */
  int32_t rx, ry;
  int64_t i0, j0;      /* global offset of this tile (tile i = 1 is global i0 + 1) */
  int64_t nx, ny;      /* tile extents */
  int32_t west, east, south, north; /* neighbour ranks or -1 */
} hfb_decomp;
/* Pure host computation (no device needed): balanced block split, remainder to the
 * leading tiles. */
hfb_status hfb_decomp_init(hfb_decomp* d);
/* Face boxes exchanged per halo update, in tile-local 1-based (i, j) coordinates:
 * for side s in {0:west,1:east,2:south,3:north} the SEND box (interior cells the
 * neighbour needs) and the RECV box (halo cells filled from it). Boxes are
 * {ilo, ihi, jlo, jhi}; empty boxes have ihi < ilo. Corners travel with the
 * north/south faces after the east/west exchange (two-phase). */
hfb_status hfb_decomp_faces(const hfb_decomp* d, int32_t side, int64_t send_box[4],
                            int64_t recv_box[4]);
/* Attach a decomposition to a context: kernels then test boundaries on GLOBAL
 * indices and stencil entries exchange halos before each stencil launch.
 * `nccl_id` is the 128-byte ncclUniqueId shared by all ranks (one process per rank), or
 * NULL when the rank will join an in-process group (hfb_group_create). */
hfb_status hfb_set_decomposition(hfb_ctx* ctx, const hfb_decomp* d, const void* nccl_id);
/* In-process rank group: contexts (ranks 0..n-1 of one decomposition, set with a NULL
 * NCCL id) driven by one host thread, halos pulled by device-to-device copies. Runs the
 * decomposed path without NCCL, e.g. several tiles on one GPU. hfb_group_run executes
 * `entry` on every rank in lockstep (main/simulation_run: copy-in on all ranks, nsteps x
 * step on every rank, copy-out). */
typedef struct hfb_group hfb_group;
hfb_status hfb_group_create(hfb_ctx* const* ctxs, int n, hfb_group** out);
void hfb_group_destroy(hfb_group* group);
hfb_status hfb_group_run(hfb_group* group, const char* entry, hfb_launch_stats* stats);
/* The device layout of a module array (include/../csrc/hfb_layout.cuh: I fastest, 128-B
 * aligned rows, a 2-cell I/J halo ring) and host twins of the halo pack/unpack kernels
 * (box {ilo, ihi, jlo, jhi} in tile-local 1-based (i, j) x all nk levels, packed i fastest,
 * then j, then k — the kernels' exact element order). `origin` is the element (1, 1, 1) of
 * a buffer in that layout. Pure host code: used by host-staged transports and by the CPU
 * multi-process tests (tests/test_decomp_gloo.py). */
hfb_status hfb_layout_of(int64_t ni, int64_t nj, int64_t nk, int64_t nl, int64_t* pitch,
                         int64_t* plane, int64_t* alloc_elems, int64_t* origin_off);
hfb_status hfb_pack_box_host(const double* origin, int64_t pitch, int64_t plane, int64_t nk,
                             const int64_t box[4], double* buf);
hfb_status hfb_unpack_box_host(double* origin, int64_t pitch, int64_t plane, int64_t nk,
                               const int64_t box[4], const double* buf);
/* halo bytes moved by this context so far (for NVLink accounting) */
int64_t hfb_halo_bytes(hfb_ctx* ctx);
/* host->device and device->host bytes transferred by this context so far */
hfb_status hfb_transfer_bytes(hfb_ctx* ctx, int64_t* h2d, int64_t* d2h);
/* 128-byte ncclUniqueId for hfb_set_decomposition (rank 0 creates, all ranks share) */
hfb_status hfb_nccl_unique_id(void* out128);
/* Peer-memory transport (one process per rank, NVLink/NVSwitch P2P; replaces NCCL for
 * the halo exchange and the reduction): after hfb_set_decomposition (NULL id) and
 * binding every array, each rank exports a blob (its device buffers' CUDA IPC handles,
 * layouts and a signal block; `buf` NULL queries the length), the caller all-gathers
 * the blobs (e.g. torch.distributed) and every rank attaches all of them. Halo updates
 * are then one push kernel storing the boundary cells straight into the neighbours'
 * halo rings (corners included, single phase) plus a release/acquire flag; reductions
 * sum the ranks' partials in rank order (deterministic). */
hfb_status hfb_peer_export(hfb_ctx* ctx, void* buf, size_t cap, size_t* len);
hfb_status hfb_peer_attach(hfb_ctx* ctx, int n, const void* const* blobs, const size_t* lens);
/* Teardown: a rank's last dycore step still stores halo cells into its neighbours'
 * buffers, so every rank must have returned from its last hfb_run / hfb_synchronize
 * (e.g. a torch.distributed barrier) before any rank calls hfb_destroy. */
/* halo updates so far: by the push kernel / handed off by the previous step's epilogue
 * (consecutive dycore steps store their edge outputs into the neighbours' halo rings) */
hfb_status hfb_peer_stats(hfb_ctx* ctx, int64_t* pushes, int64_t* handoffs);

/* --- reductions (reduction.h90 `reduce(+:total)`) ---------------------------------- */
/* 0 (default): fast two-level tree sum, equal to the reference to 1e-12 relative
 * (SPEC.md:473). 1: ordered — the reference's acc-simulated order (interp.cpp:1080-1173):
 * one partial per (i,j) iteration summing k = 1..nz from the identity, combined in
 * linear-id order (i fastest) starting from the initial value, i.e. bit-identical to
 * run_gpu_simulated on the OpenACC backend. Ordered runs single-domain, in an
 * in-process group, or one process per rank over the peer transport (the tiles' column
 * partials are assembled in global order on every rank). */
hfb_status hfb_set_reduction_order(hfb_ctx* ctx, int ordered);

/* --- per-context options (explicit; the library reads no environment variables) ------
 * "variant": which kernels run the dycore steps — "product" (default: the fused
 *   warp-specialised step), "generic" (portable kernels), "split" (advect + acoustic
 *   kernels), "single_role" (fused, one role per warp); "tma" and "ws2" (measured-slower
 *   alternatives) exist only in the A/B build libhfb_variants.so, elsewhere HFB_CONFIG.
 * "arith": "exact" (default, bit-identical to the reference's binary64 evaluation) or
 *   "fma" (the fused step compiled with FMA contraction; within 1e-12 relative per field
 *   after one step, tests/test_gpu_tolerance.py).
 * "checked": "1" tracks element init flags on the device (see hfb_bind_init) — the
 *   debug mode in which programs generated with `hfc --checked` also check every array
 *   access against the declared bounds (interp.cpp:487-492).
 * "overlap": "1" (default) overlaps the halo exchange with the interior columns, "0"
 *   serialises (both orders are bit-identical).
 * "debug_skip": A/B build only, timing experiments (1 = no advection, 2 = no acoustic).
 * Every variant gives bit-identical results. */
hfb_status hfb_set_option(hfb_ctx* ctx, const char* key, const char* value);
/* 1 in the A/B build (libhfb_variants.so), 0 in the product library */
int hfb_variants_build(void);

/* --- state images and scenario files ------------------ */
/* HFBSTAT1 image of the context's MachineState: program, every scalar (with its set
 * flag), every bound array in the reference's ArrayValue order (row-major, last subscript
 * fastest, interp.cpp:485-494; independent of device layout and host order), FNV-1a
 * trailer. Arrays whose device copy is newer are read back without changing residency.
 * The format is documented in csrc/hfb_runtime.cu and mirrored by state.py. */
hfb_status hfb_save_state(hfb_ctx* ctx, const char* path);
/* Restore an image (checkpoint/resume): loads the program when none is loaded (else it
 * must match), sets every scalar, and writes every array into its bound host buffer
 * (same bounds required) or into a context-owned pinned buffer it binds. Restored arrays
 * are host-newer (a later copy-in transfers them). A corrupt image is HFB_IO. */
hfb_status hfb_load_state(hfb_ctx* ctx, const char* path);
/* the host buffer bound to an array (the caller's or a context-owned one), its bounds and
 * element strides per dim (unused dims: bounds 1, stride 0) */
hfb_status hfb_host_array(hfb_ctx* ctx, const char* module, const char* name, double** host,
                          int* rank, int64_t lower[4], int64_t upper[4], int64_t strides[4]);
/* checksums of an array's newest copy in ArrayValue order: the fp64 sum in that order
 * and the FNV-1a 64 hash of its raw little-endian bytes (either output may be NULL) */
hfb_status hfb_array_checksum(hfb_ctx* ctx, const char* module, const char* name, double* sum,
                              uint64_t* bits);
/* Scenario file (text; the reference's harness input): `program`, `entry`,
 * `set` scalars, optional `array` bounds, `fill` patterns (const v | ramp a b |
 * splitmix seed offset scale, the reference SplitMix64 over the ArrayValue flat index,
 * interp.cpp:22-28) and `expect` checksums (array sum value rel_tol | array bits hex |
 * scalar value v rel_tol). Filled arrays are bound to context-owned buffers (or the
 * caller's, if bound with the same bounds), the entry runs, then every expectation is
 * checked: HFB_VALIDATION names the first that fails. `report` (may be NULL) receives one
 * line per expectation. */
hfb_status hfb_run_scenario(hfb_ctx* ctx, const char* path, hfb_launch_stats* stats,
                            char* report, size_t report_len);

/* --- measurement --------------------------------------------------------------------- */
/* enable (1) / disable (0) CUDA-event timing of every native launch on the context
 * stream; -1 also clears the accumulated times */
hfb_status hfb_profile(hfb_ctx* ctx, int enable);
/* accumulated device time and launch count of one native kernel ("dycore_advect",
 * "dycore_acoustic", "hfk0_diffuse_step", ...); synchronises on the pending events */
hfb_status hfb_kernel_time(hfb_ctx* ctx, const char* kernel, double* total_ms, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* HFB_H */
