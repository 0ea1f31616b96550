/* hfb_plugin.h — ABI between libhfb.so and programs compiled from Hybrid-Fortran sources
 * by the code generator (paper_1710_08616_b200/hfc).
 *
 * The reference's backend turns a `.h90` program into CUDA-Fortran text
 * (codegen.cpp:397-519: host wrappers hfd_<routine>, kernels hfk<i>_<routine>). Here the
 * generator emits CUDA C++ for sm_100a, nvcc builds it into a shared object, and
 * hfb_load_program(ctx, "<path>.so") loads it: the context then holds that program's
 * module state (scalars, arrays in the engine's device layout) exactly as it holds a
 * built-in app's, and hfb_run(ctx, entry, ...) runs the generated host driver.
 */
#ifndef HFB_PLUGIN_H
#define HFB_PLUGIN_H

#include <stdint.h>

#include "hfb.h"

#ifdef __cplusplus
extern "C" {
#endif

#define HFB_PLUGIN_ABI 1

typedef struct {
  const char* name;
  int type; /* 0 integer(4), 1 real(r_size), 2 logical */
} hfb_plugin_scalar;

typedef struct {
  const char* name;
  int rank;
  const char* lower[4]; /* literal or module scalar name, per dim */
  const char* upper[4];
  int roles[4];         /* 0 I, 1 J, 2 K, 3 L: the device storage order of each dim */
} hfb_plugin_array;

typedef struct {
  int abi; /* HFB_PLUGIN_ABI */
  const char* program;
  const char* module;                 /* the state module */
  const hfb_plugin_scalar* scalars;   /* terminated by name == NULL */
  const hfb_plugin_array* arrays;     /* terminated by name == NULL */
  const char* const* entries;         /* host routines, NULL-terminated */
  const char* const* transfer_entries; /* entries that perform host transfers */
  /* run a host routine; stats accumulate; returns an hfb_status */
  int (*run)(hfb_ctx* ctx, const char* routine, hfb_launch_stats* stats, int allow_transfers);
} hfb_plugin_desc;

/* the one symbol a program plugin exports */
const hfb_plugin_desc* hfb_plugin(void);

/* --- services libhfb.so provides to generated code -------------------------------- */
/* device view of an array: element(d0..) = origin[sum (d - lower[d]) * stride[d]] */
typedef struct {
  double* origin;
  int64_t stride[4];
  int64_t lower[4];
} hfb_view;
/* residency checks before a kernel reads (mode 0) or reads and writes (mode 2) a module
 * array (interp.cpp:397-411); routine-local (scratch) arrays always pass */
hfb_status hfb_plugin_prepare(hfb_ctx* ctx, const char* name, int mode);
/* a kernel wrote the array: the device copy is the newest (interp.cpp:533-538) */
hfb_status hfb_plugin_written(hfb_ctx* ctx, const char* name);
/* device view of a module array (allocated on first use) or of a scratch array */
hfb_status hfb_plugin_view(hfb_ctx* ctx, const char* name, hfb_view* out);
/* host view of a module array's bound host buffer for host-code element access (the
 * generated host drivers); reads of a host copy older than the device copy fail, writes
 * make the host copy the newest (interp.cpp:406-409) */
hfb_status hfb_plugin_host(hfb_ctx* ctx, const char* name, int write, hfb_view* out);
/* the same without a call per element: the host view plus the array's residency word
 * (0 host newer, 1 device newer, 2 both equal) and its has-a-device-copy flag; generated
 * host code checks a read against residency 1 (then calls hfb_plugin_host for the
 * error) and sets residency 0 on a write when a device copy exists — slot_side's rules */
typedef struct {
  hfb_view view;
  int32_t* residency;
  const int32_t* has_device;
} hfb_host_ref;
hfb_status hfb_plugin_host_ref(hfb_ctx* ctx, const char* name, hfb_host_ref* out);
/* context-owned device scratch array `key` (a routine-local array, possibly extended by
 * the region domain; analysis.cpp:439-527), (re)allocated when its bounds change */
hfb_status hfb_plugin_scratch(hfb_ctx* ctx, const char* key, int rank, const int64_t* lower,
                              const int64_t* upper, const int* roles);

/* --- checked mode (programs generated with `hfc --checked`) ------------------------- */
/* Declared bounds and element init flags of a module or scratch array, for the checked
 * accessors: `dinit` (device, one byte per element at the data's element offsets
 * relative to hfb_view.origin) and `hinit` (the caller's host flags bound with
 * hfb_bind_init, at the host buffer's offsets; NULL if none). Module arrays whose init
 * flags were never tracked count as fully set. */
hfb_status hfb_plugin_array_info(hfb_ctx* ctx, const char* name, int* rank, int64_t lower[4],
                                 int64_t upper[4], uint8_t** dinit, uint8_t** hinit);
/* a routine-local array starts every routine invocation with no element set
 * (elaborate_locals, interp.cpp:936-979) */
hfb_status hfb_plugin_scratch_clear_init(hfb_ctx* ctx, const char* key);
/* fail the current run with `status` and the message (the reference's texts) */
hfb_status hfb_plugin_error(hfb_ctx* ctx, hfb_status status, const char* msg);

#ifdef __cplusplus
}
#endif
#endif /* HFB_PLUGIN_H */
