// hfb_runtime.cu — host runtime behind include/hfb.h.
//
// Plays the part of the reference's executor for GPU programs
// (/root/reference/proj/src/interp.cpp: Executor::exec_transfer :1369-1415,
// exec_launch :1417-1475, slot_side residency :397-411) but runs native sm_100a
// kernels instead of interpreting the generated CUDA-Fortran: a context holds the
// MachineState-equivalent (module scalars + caller-owned host buffers), the device
// copies in the I-fastest layout (hfb_layout.cuh), the residency state machine, and
// the app programs, whose entries follow the generated host code
// (transfers at `transferHere` routines, codegen.cpp:570-600; kernel launches per
// @parallelRegion, codegen.cpp:397-449).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/hfb.h"
#include "../../include/hfb_plugin.h"
#include "hfb_kernels.cuh"
#include "hfb_layout.cuh"

namespace {
// NVTX ranges (header-only NVTX3: free unless a tool such as ncu/nsys is attached): one
// per native launch, entry, transfer and halo update (SURVEY §5 tracing)
struct NvtxRange {
  explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

using namespace hfb;

namespace {

thread_local std::string g_last_error = "";

// An hft::Error analogue: kind (status) + message.
struct Fail {
  hfb_status code;
  std::string msg;
};

[[noreturn]] void fail(hfb_status code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw Fail{code, buf};
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(HFB_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

std::string lower(const char* s) {
  std::string r = s ? s : "";
  for (char& c : r) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return r;
}

template <class F>
hfb_status guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return HFB_OK;
  } catch (const Fail& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return HFB_RUNTIME;
  }
}

// ---------------------------------------------------------------------------
// Program description: the built-in apps' modules (declarations as in the .h90)
// ---------------------------------------------------------------------------
enum class SType { Int, Real };

struct ScalarDecl {
  std::string name;
  SType type;
  bool is_param = false;
  double param = 0.0;
};

struct ArrayDecl {
  std::string name;
  std::vector<std::pair<std::string, std::string>> dims;  // (lower expr, upper expr)
  std::vector<Role> roles;
  bool pingpong = false;  // state array the timestep rewrites in full (double-buffered)
};

struct AppDecl {
  std::string app, module;
  std::vector<ScalarDecl> scalars;
  std::vector<ArrayDecl> arrays;
  const hfb_plugin_desc* plugin = nullptr;  // generated program (include/hfb_plugin.h)
};

std::vector<std::pair<std::string, std::string>> dims3(const char* a, const char* b,
                                                       const char* c) {
  return {{"1", a}, {"1", b}, {"1", c}};
}

const std::vector<AppDecl>& app_table() {
  static const std::vector<AppDecl> apps = [] {
    std::vector<AppDecl> v;
    const std::vector<Role> KIJ = {kRoleK, kRoleI, kRoleJ};
    const std::vector<Role> IJ = {kRoleI, kRoleJ};
    // diffusion.h90:1-10
    v.push_back({"diffusion",
                 "diff_state",
                 {{"nx", SType::Int}, {"ny", SType::Int}, {"nz", SType::Int},
                  {"nsteps", SType::Int}, {"coef", SType::Real}},
                 {{"t_old", dims3("nz", "nx", "ny"), KIJ, true},
                  {"t_new", dims3("nz", "nx", "ny"), KIJ, false}}});
    // damping.h90:1-14
    {
      std::vector<std::pair<std::string, std::string>> d3 = {
          {"nz_mn", "nz_mx"}, {"nx_mn", "nx_mx"}, {"ny_mn", "ny_mx"}};
      auto d4 = d3;
      d4.push_back({"1", "2"});
      v.push_back({"damping",
                   "svar",
                   {{"nx_mn", SType::Int}, {"nx_mx", SType::Int}, {"ny_mn", SType::Int},
                    {"ny_mx", SType::Int}, {"nz_mn", SType::Int}, {"nz_mx", SType::Int},
                    {"tratio_bnd", SType::Real}, {"mtratio_bnd", SType::Real}},
                   {{"dens_ref_f", d3, KIJ},
                    {"dens_ptb_damp", d3, KIJ},
                    {"dens_ptb_bnd", d4, {kRoleK, kRoleI, kRoleJ, kRoleL}}}});
    }
    // bounded.h90:1-7
    v.push_back({"bounded",
                 "b_state",
                 {{"nx", SType::Int}, {"ny", SType::Int}},
                 {{"a", {{"1", "nx"}, {"1", "ny"}}, IJ}, {"b", {{"1", "nx"}, {"1", "ny"}}, IJ}}});
    // sf_state.h90:1-11 (cover_frac's tile dim rides the K role)
    v.push_back({"surface_flux",
                 "sf_state",
                 {{"ntlm", SType::Int, true, 4.0},
                  {"nx", SType::Int},
                  {"ny", SType::Int},
                  {"tile_land", SType::Int}},
                 {{"cover_frac", dims3("ntlm", "nx", "ny"), KIJ},
                  {"wind_speed", {{"1", "nx"}, {"1", "ny"}}, IJ},
                  {"flx_sum_x", {{"1", "nx"}, {"1", "ny"}}, IJ},
                  {"flx_sum_y", {{"1", "nx"}, {"1", "ny"}}, IJ}}});
    // reduction.h90:1-8
    v.push_back({"reduction",
                 "red_state",
                 {{"nx", SType::Int}, {"ny", SType::Int}, {"nz", SType::Int},
                  {"total", SType::Real}},
                 {{"y", dims3("nz", "nx", "ny"), KIJ}}});
    // apps/dycore/dyn_state.h90
    v.push_back({"dycore",
                 "dyn_state",
                 {{"nx", SType::Int}, {"ny", SType::Int}, {"nz", SType::Int},
                  {"nsteps", SType::Int}, {"dt", SType::Real}, {"rdx", SType::Real},
                  {"rdy", SType::Real}, {"rdz", SType::Real}, {"cs2", SType::Real},
                  {"grav", SType::Real}, {"th0", SType::Real}, {"ch", SType::Real},
                  {"rrelax", SType::Real}, {"nsound", SType::Int}, {"nbnd", SType::Int},
                  {"kdmp", SType::Int}, {"rdmp", SType::Real}, {"rnbnd", SType::Real},
                  {"rnzd", SType::Real}},
                 {{"rho", dims3("nz", "nx", "ny"), KIJ, false},
                  {"th", dims3("nz", "nx", "ny"), KIJ, true},
                  {"u", dims3("nz", "nx", "ny"), KIJ, true},
                  {"v", dims3("nz", "nx", "ny"), KIJ, true},
                  {"w", dims3("nz", "nx", "ny"), KIJ, true},
                  {"p", dims3("nz", "nx", "ny"), KIJ, true},
                  {"tsfc", {{"1", "nx"}, {"1", "ny"}}, IJ, false},
                  {"colm", {{"1", "nx"}, {"1", "ny"}}, IJ, false}}});
    return v;
  }();
  return apps;
}

// ---------------------------------------------------------------------------
// State
// ---------------------------------------------------------------------------
enum Residency : int32_t { kHost = 0, kDevice = 1, kBoth = 2 };  // interp.hpp:30

struct Scalar {
  SType type;
  int64_t i = 0;
  double r = 0.0;
  bool init = false;
};

struct Slot {
  std::string module, name;
  const ArrayDecl* decl = nullptr;
  // host side (caller-owned)
  double* host = nullptr;
  int rank = 0;
  int64_t lower[4] = {1, 1, 1, 1}, upper[4] = {1, 1, 1, 1}, hstride[4] = {0, 0, 0, 0};
  int64_t count = 0;
  bool pinned = false;
  double* owned = nullptr;  // context-owned host buffer (hfb_load_state / scenarios)
  // device side
  Layout lay;
  double* dev[3] = {nullptr, nullptr, nullptr};  // [2] only for RK3 stage states
  int cur = 0;
  int32_t has_device = 0;  // a device copy exists (bool; int32 for hfb_plugin_host_ref)
  // element init flags (ArrayValue::init, interp.hpp:16-28): the caller's, at the host
  // buffer's element offsets (hfb_bind_init), and the device copy's, one byte per element
  // in the device layout (kept while the context tracks init: checked mode or bound flags)
  uint8_t* hinit = nullptr;
  uint8_t* dinit = nullptr;
  Residency res = kHost;
  cudaStream_t stream = nullptr;  // owning context's stream

  double* d() const { return dev[cur] + lay.origin_off; }
  int alt() const { return cur == 0 ? 1 : 0; }
  double* d_alt() const { return dev[alt()] + lay.origin_off; }
  double* d_buf(int b) const { return dev[b] + lay.origin_off; }
};

}  // namespace

struct hfb_group {
  std::vector<hfb_ctx*> ranks;
};

namespace {
// peer-memory transport: a neighbour's field buffers and signal block, mapped into this
// process by CUDA IPC (hfb_peer_attach)
struct PeerField {
  double* base[3] = {nullptr, nullptr, nullptr};
  int nbuf = 0;
  int64_t pitch = 0, plane = 0, origin_off = 0;
};
struct PeerRank {
  int64_t nx = 0, ny = 0;
  uint64_t* sig = nullptr;
  double* gather = nullptr;  // 2 x global_nx x global_ny: ordered-reduction partials
  std::map<std::string, PeerField> fields;
};
// signal block layout (uint64 words): [0, 9) halo flags by the sender's offset from the
// receiver, [16, 80) reduction flags by sender rank, then 2 x 64 doubles of reduction
// slots (parity of the reduction epoch)
// signal block words: halo flags per neighbour direction (0..8), this rank's halo epoch
// counter (9, device side: graph replays advance it), reduction flags, reduction slots
constexpr int kSigHalo = 0, kSigEpoch = 9, kSigRed = 16, kSigSlots = 80, kSigWords = 80 + 128;
// device scratch of generated programs: routine-local arrays (hfb_plugin_scratch)
struct Scratch {
  Layout lay;
  double* dev = nullptr;
  uint8_t* dinit = nullptr;  // checked generated programs: element init flags
  int rank = 0;
  int64_t lower[4] = {1, 1, 1, 1}, upper[4] = {1, 1, 1, 1};
  Role roles[4] = {kRoleI, kRoleJ, kRoleK, kRoleL};
};
}  // namespace

struct hfb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  const AppDecl* app = nullptr;
  std::map<std::string, Scalar> scalars;  // key: name (single module per app)
  std::map<std::string, Slot> slots;
  double* staging = nullptr;
  size_t staging_bytes = 0;
  double* red_partials = nullptr;
  double* red_result = nullptr;
  double* red_host = nullptr;
  hfb_decomp decomp{};
  bool decomposed = false;
  // in-process rank group (all ranks' contexts driven by one host thread; halos are
  // pulled by device copies instead of NCCL): used to exercise the decomposed path
  // bit-for-bit on a single GPU
  struct hfb_group* group = nullptr;
  int64_t steps_done = 0;    // per-step entries completed (pull-side buffer selection)
  double red_local = 0.0;    // this rank's partial of a group reduction
  // ordered reductions (hfb_set_reduction_order): per-column partials of this tile
  bool reduce_ordered = false;
  double* red_cols = nullptr;
  size_t red_cols_cap = 0;
  int64_t halo_bytes = 0;
  int64_t h2d_bytes = 0, d2h_bytes = 0;  // host <-> device transfer bytes (hfb_transfer_bytes)
  // NCCL (multi-process decomposition)
  void* nccl_comm = nullptr;
  double* halo_send = nullptr;
  double* halo_recv = nullptr;
  size_t halo_cap = 0;
  std::map<std::string, Scratch> scratch;  // generated programs' routine-local arrays
  // asuca_step: the stage's slow tendencies (frho, fth, fu, fv, fw) and the RK2 midpoint
  // pressure pa, in the prognostic fields' device layout
  double* asu[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int64_t asu_elems = 0;
  bool asu_exported = false;  // fu, fv, pa are mapped by the peers (hfb_peer_export)
  // peer-memory halo transport (hfb_peer_export / hfb_peer_attach): halos are stored
  // straight into the neighbours' buffers over NVLink, flags signal their arrival
  bool peer = false;
  // the current buffers' halo rings were stored by the neighbours' previous step (fused
  // remote epilogue): the next exchange only waits for their flags
  bool peer_fused = false;
  int64_t peer_pushes = 0, peer_handoffs = 0;  // exchanges by push kernel / by epilogue
  uint64_t* peer_sig = nullptr;
  double* peer_gather = nullptr;  // this rank's gather buffer (ordered reductions)
  uint64_t halo_epoch = 0, red_epoch = 0;
  std::vector<PeerRank> peers;
  std::vector<void*> ipc_opened;
  // halo exchange overlapped with the interior columns (decomposed stencil steps): the
  // exchange runs on `comm` while the columns that never read the halo ring run on
  // `stream`; the boundary strips follow the exchange (hfb_set_option "overlap" "0" serialises)
  cudaStream_t comm = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
  // the stream step kernels go to (nullptr: `stream`); exchange_and_run points it at
  // `comm` for the boundary strips, which then overlap the interior launch
  cudaStream_t run_stream = nullptr;
  bool overlap = true;  // hfb_set_option(ctx, "overlap", "0") serialises
  // CUDA graph cache for hfb_run_graph
  // CUDA graphs of captured step sequences (hfb_run_graph / hfb_enqueue_graph), keyed by
  // entry, step count, the buffer sides at the start and the peer hand-off state
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    hfb_launch_stats stats{};
    std::map<std::string, int> cur1;  // buffer sides after the steps
    bool peer_fused1 = false;         // peer hand-off state after the steps
    int64_t pushes = 0, handoffs = 0, halo_bytes = 0, epochs = 0;  // per replay
  };
  std::map<std::string, GraphEntry> graphs;
  // kernel variant (hfb_set_option "variant"; explicit per context, never from the
  // environment): the portable kernels only / the two-kernel (advect + acoustic) split /
  // the single-role fused kernel; tma / ws2 exist only in the A/B build (make variants)
  bool force_generic = false;
  bool force_split = false;
  bool force_single_role = false;
  bool force_tma = false;
  bool force_ws2 = false;
  int debug_skip = 0;  // A/B build only: 1 = no advection, 2 = no acoustic (timing)
  // hfb_set_option "arith": the fused step's FMA-contracted build (tolerance mode)
  bool arith_fma = false;
  // hfb_set_option "checked": track element init flags on the device and check reads
  // (the reference's unset-read and bounds errors, interp.cpp:487-507)
  bool checked = false;
  int* chk_flag = nullptr;  // device word of the init-box checks
  bool plugin_tracks_init = false;  // the loaded program is a checked build (hfc --checked)
  // per-kernel CUDA-event timing (hfb_profile)
  bool prof = false;
  bool capturing = false;
  struct Timed {
    std::string name;
    cudaEvent_t a, b;
  };
  std::vector<Timed> pending;
  std::vector<cudaEvent_t> free_events;
  std::map<std::string, std::pair<double, int64_t>> kernel_ms;  // name -> (ms, launches)
};

namespace {

// ---------------------------------------------------------------------------
// small helpers on the context
// ---------------------------------------------------------------------------
Scalar& scalar_ref(hfb_ctx* c, const std::string& module, const std::string& name) {
  if (!c->app) fail(HFB_CONFIG, "no program loaded (hfb_load_program)");
  if (module != c->app->module)
    fail(HFB_CONFIG, "unknown module '%s' (program '%s' has module '%s')", module.c_str(),
         c->app->app.c_str(), c->app->module.c_str());
  auto it = c->scalars.find(name);
  if (it == c->scalars.end())
    fail(HFB_CONFIG, "'%s' is not a scalar of module '%s'", name.c_str(), module.c_str());
  return it->second;
}

int64_t ival(hfb_ctx* c, const char* name) {
  auto it = c->scalars.find(name);
  if (it == c->scalars.end() || !it->second.init)
    fail(HFB_RUNTIME, "read of unset variable '%s'", name);  // interp.cpp:549
  return it->second.type == SType::Int ? it->second.i : static_cast<int64_t>(it->second.r);
}

double rval(hfb_ctx* c, const char* name) {
  auto it = c->scalars.find(name);
  if (it == c->scalars.end() || !it->second.init)
    fail(HFB_RUNTIME, "read of unset variable '%s'", name);
  return it->second.type == SType::Real ? it->second.r : static_cast<double>(it->second.i);
}

int64_t eval_dim(hfb_ctx* c, const std::string& e) {
  if (!e.empty() && (std::isdigit(static_cast<unsigned char>(e[0])) || e[0] == '-'))
    return std::stoll(e);
  return ival(c, e.c_str());
}

Slot& slot_ref(hfb_ctx* c, const std::string& module, const std::string& name) {
  if (!c->app) fail(HFB_CONFIG, "no program loaded (hfb_load_program)");
  if (module != c->app->module)
    fail(HFB_CONFIG, "unknown module '%s'", module.c_str());
  auto it = c->slots.find(name);
  if (it == c->slots.end())
    fail(HFB_CONFIG, "'%s' is not an array of module '%s'", name.c_str(), module.c_str());
  return it->second;
}

Slot& slot(hfb_ctx* c, const char* name) { return slot_ref(c, c->app->module, name); }

// declared bounds vs the bound buffer
void check_bounds(hfb_ctx* c, Slot& s) {
  if (!s.host) fail(HFB_CONFIG, "array '%s' of module '%s' is not bound", s.name.c_str(),
                    s.module.c_str());
  for (size_t d = 0; d < s.decl->dims.size(); ++d) {
    int64_t lo = eval_dim(c, s.decl->dims[d].first), hi = eval_dim(c, s.decl->dims[d].second);
    if (lo != s.lower[d] || hi != s.upper[d])
      fail(HFB_RUNTIME,
           "array '%s' is bound with bounds [%lld:%lld] in dimension %zu but declared "
           "[%lld:%lld]",
           s.name.c_str(), (long long)s.lower[d], (long long)s.upper[d], d + 1, (long long)lo,
           (long long)hi);
  }
}

void role_extents(const Slot& s, int64_t ext[4], int64_t hs[4]) {
  for (int r = 0; r < 4; ++r) {
    ext[r] = 1;
    hs[r] = 0;
  }
  for (int d = 0; d < s.rank; ++d) {
    Role r = s.decl->roles[d];
    ext[r] = s.upper[d] - s.lower[d] + 1;
    hs[r] = s.hstride[d];
  }
}

void ensure_device(hfb_ctx* c, Slot& s, bool second, int nbuf = 0) {
  if (!s.dev[0]) {
    int64_t ext[4], hs[4];
    role_extents(s, ext, hs);
    s.lay = Layout::make(ext[kRoleI], ext[kRoleJ], ext[kRoleK], ext[kRoleL]);
  }
  const int want = nbuf ? nbuf : (second ? 2 : 1);
  for (int b = 0; b < want; ++b) {
    if (s.dev[b]) continue;
    size_t bytes = static_cast<size_t>(s.lay.alloc_elems) * sizeof(double);
    cuda_check(cudaMalloc(&s.dev[b], bytes), "cudaMalloc(device array)");
    cuda_check(cudaMemsetAsync(s.dev[b], 0, bytes, c->stream), "cudaMemsetAsync");
  }
}

void ensure_staging(hfb_ctx* c, size_t bytes) {
  if (c->staging_bytes >= bytes) return;
  if (c->staging) cudaFree(c->staging);
  c->staging = nullptr;
  cuda_check(cudaMalloc(&c->staging, bytes), "cudaMalloc(staging)");
  c->staging_bytes = bytes;
}

Relayout relayout_of(const Slot& s) {
  Relayout r{};
  role_extents(s, r.ext, r.hs);
  r.ds[kRoleI] = 1;
  r.ds[kRoleJ] = s.lay.pitch;
  r.ds[kRoleK] = s.lay.plane;
  r.ds[kRoleL] = s.lay.volume;
  r.fast = kRoleI;
  for (int role = 0; role < 4; ++role)
    if (r.hs[role] == 1 && r.ext[role] > 1) r.fast = role;
  if (r.hs[kRoleI] == 1 || r.ext[kRoleI] == 1) {
    // keep I as the copy axis when it is host-contiguous (or trivially so)
    if (r.hs[kRoleI] == 1) r.fast = kRoleI;
  }
  if (r.fast != kRoleI && r.ext[r.fast] <= 1) r.fast = kRoleI;
  return r;
}

// ---------------------------------------------------------------------------
// transfers (interp.cpp:1369-1415)
// ---------------------------------------------------------------------------
// ---- element init flags (checked mode / bound flags) -------------------------------
bool tracks_init(const hfb_ctx* c, const Slot& s) { return c->checked || s.hinit; }

void ensure_dinit(hfb_ctx* c, Slot& s, int fill) {
  if (s.dinit) return;
  cuda_check(cudaMalloc(&s.dinit, static_cast<size_t>(s.lay.alloc_elems)), "cudaMalloc(init)");
  cuda_check(cudaMemsetAsync(s.dinit, fill, static_cast<size_t>(s.lay.alloc_elems), c->stream),
             "cudaMemsetAsync(init)");
}

// the device copy's init flags := the bound host flags (copy-in) / all set / all clear
void dinit_upload(hfb_ctx* c, Slot& s) {
  ensure_dinit(c, s, 1);
  if (!s.hinit) {
    cuda_check(cudaMemsetAsync(s.dinit, 1, static_cast<size_t>(s.lay.alloc_elems), c->stream),
               "cudaMemsetAsync(init)");
    return;
  }
  ensure_staging(c, static_cast<size_t>(s.count) * sizeof(double));
  uint8_t* st = reinterpret_cast<uint8_t*>(c->staging);
  cuda_check(cudaMemcpyAsync(st, s.hinit, static_cast<size_t>(s.count), cudaMemcpyHostToDevice,
                             c->stream),
             "cudaMemcpyAsync(init H2D)");
  cuda_check(launch_relayout_u8(st, s.dinit + s.lay.origin_off, relayout_of(s), true, c->stream),
             "relayout(init H2D)");
}

void dinit_download(hfb_ctx* c, Slot& s) {
  if (!s.hinit || !s.dinit) return;
  ensure_staging(c, static_cast<size_t>(s.count) * sizeof(double));
  uint8_t* st = reinterpret_cast<uint8_t*>(c->staging);
  cuda_check(launch_relayout_u8(s.dinit + s.lay.origin_off, st, relayout_of(s), false, c->stream),
             "relayout(init D2H)");
  cuda_check(cudaMemcpyAsync(s.hinit, st, static_cast<size_t>(s.count), cudaMemcpyDeviceToHost,
                             c->stream),
             "cudaMemcpyAsync(init D2H)");
  cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
}

// A built-in kernel reads / writes the elements of `s` within declared bounds [lo, hi]
// (per declared dim; NULL = the whole array). Reads of an unset element fail with the
// reference's text (interp.cpp:505-507); writes set the flags (write_element, :534).
InitBox init_box(const Slot& s, const int64_t* lo, const int64_t* hi) {
  InitBox b{};
  for (int r = 0; r < 4; ++r) {
    b.lo[r] = 0;
    b.n[r] = 1;
  }
  b.ds[kRoleI] = 1;
  b.ds[kRoleJ] = s.lay.pitch;
  b.ds[kRoleK] = s.lay.plane;
  b.ds[kRoleL] = s.lay.volume;
  for (int d = 0; d < s.rank; ++d) {
    const Role r = s.decl->roles[d];
    const int64_t l = lo ? lo[d] : s.lower[d], h = hi ? hi[d] : s.upper[d];
    b.lo[r] = l - s.lower[d];
    b.n[r] = h - l + 1;
  }
  return b;
}

void init_read(hfb_ctx* c, const char* name, const int64_t* lo = nullptr,
               const int64_t* hi = nullptr) {
  Slot& s = slot(c, name);
  if (!s.dinit) return;  // not tracked: the contents count as defined
  if (!c->chk_flag) cuda_check(cudaMalloc(&c->chk_flag, sizeof(int)), "cudaMalloc(flag)");
  cuda_check(cudaMemsetAsync(c->chk_flag, 0, sizeof(int), c->stream), "cudaMemsetAsync");
  const InitBox b = init_box(s, lo, hi);
  for (int q = 0; q < 4; ++q)
    if (b.n[q] <= 0) return;
  cuda_check(launch_init_box(s.dinit + s.lay.origin_off, b, 0, c->chk_flag, c->stream),
             "init check");
  int flag = 0;
  cuda_check(cudaMemcpyAsync(&flag, c->chk_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream),
             "cudaMemcpyAsync(flag)");
  cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  if (flag) fail(HFB_RUNTIME, "read of unset element of '%s'", name);
}

void init_written(hfb_ctx* c, const char* name, const int64_t* lo = nullptr,
                  const int64_t* hi = nullptr) {
  Slot& s = slot(c, name);
  if (!s.dinit) return;
  const InitBox b = init_box(s, lo, hi);
  for (int q = 0; q < 4; ++q)
    if (b.n[q] <= 0) return;
  cuda_check(launch_init_box(s.dinit + s.lay.origin_off, b, 1, nullptr, c->stream), "init set");
}

// every array element a prognostic read touches except the upper wall plane of one dim
// (u(nx), v(ny), w(nz) of the C-grid are never read)
void init_read_but_last(hfb_ctx* c, const char* name, int dim) {
  Slot& s = slot(c, name);
  if (!s.dinit) return;
  int64_t lo[4], hi[4];
  for (int d = 0; d < s.rank; ++d) {
    lo[d] = s.lower[d];
    hi[d] = s.upper[d] - (d == dim ? 1 : 0);
  }
  init_read(c, name, lo, hi);
}

void do_device_allocate(hfb_ctx* c, Slot& s) {
  check_bounds(c, s);
  if (!s.has_device) {
    ensure_device(c, s, false);
    s.has_device = true;  // init flags cleared: contents undefined until written
    if (tracks_init(c, s)) {
      ensure_dinit(c, s, 0);
      cuda_check(cudaMemsetAsync(s.dinit, 0, static_cast<size_t>(s.lay.alloc_elems), c->stream),
                 "cudaMemsetAsync(init)");
    }
  }
}

void do_copy_to_device(hfb_ctx* c, Slot& s) {
  NvtxRange nr("hfrt_copy_to_device");
  check_bounds(c, s);
  c->peer_fused = false;
  if (s.res == kDevice)
    fail(HFB_RESIDENCY, "copy-in of '%s' would overwrite newer device data", s.name.c_str());
  ensure_device(c, s, false);
  size_t bytes = static_cast<size_t>(s.count) * sizeof(double);
  ensure_staging(c, bytes);
  cuda_check(cudaMemcpyAsync(c->staging, s.host, bytes, cudaMemcpyHostToDevice, c->stream),
             "cudaMemcpyAsync(H2D)");
  c->h2d_bytes += static_cast<int64_t>(bytes);
  cuda_check(launch_relayout(c->staging, s.d(), relayout_of(s), true, c->stream),
             "relayout(H2D)");
  if (tracks_init(c, s)) dinit_upload(c, s);  // after the data: the staging is reused
  s.has_device = true;
  s.res = kBoth;
}

void do_copy_from_device(hfb_ctx* c, Slot& s) {
  NvtxRange nr("hfrt_copy_from_device");
  if (!s.has_device)
    fail(HFB_RESIDENCY, "copy-out of '%s', which was never transferred to the device",
         s.name.c_str());
  if (s.res == kHost)
    fail(HFB_RESIDENCY, "copy-out of '%s' would overwrite newer host data", s.name.c_str());
  size_t bytes = static_cast<size_t>(s.count) * sizeof(double);
  ensure_staging(c, bytes);
  cuda_check(launch_relayout(s.d(), c->staging, relayout_of(s), false, c->stream),
             "relayout(D2H)");
  cuda_check(cudaMemcpyAsync(s.host, c->staging, bytes, cudaMemcpyDeviceToHost, c->stream),
             "cudaMemcpyAsync(D2H)");
  cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  c->d2h_bytes += static_cast<int64_t>(bytes);
  dinit_download(c, s);
  s.res = kBoth;
}

// The copy-out at the end of an entry that copied the array in itself (transferHere,
// codegen.cpp:570-600): an array the entry never wrote on the device — residency still
// Both since that copy-in — already equals its host copy inside this synchronous call,
// so the transfer is skipped (same bytes, same residency; e.g. the dycore's rho)
void entry_copy_out(hfb_ctx* c, Slot& s) {
  if (s.has_device && s.res == kBoth) return;
  do_copy_from_device(c, s);
}

// device-code access checks (slot_side, interp.cpp:397-411)
void dev_read(hfb_ctx* c, const char* name) {
  Slot& s = slot(c, name);
  if (!s.has_device)
    fail(HFB_RESIDENCY, "array '%s' has no device copy (missing transfer)", name);
  if (s.res == kHost)
    fail(HFB_RESIDENCY, "device copy of '%s' is stale (host copy was modified)", name);
}
void dev_write(hfb_ctx* c, const char* name) {
  Slot& s = slot(c, name);
  if (!s.has_device)
    fail(HFB_RESIDENCY, "array '%s' has no device copy (missing transfer)", name);
}
void dev_written(hfb_ctx* c, const char* name) { slot(c, name).res = kDevice; }

// ---------------------------------------------------------------------------
// launch contract accounting (codegen.cpp:421-434; interp.cpp:1417-1475)
// ---------------------------------------------------------------------------
struct Stats {
  int64_t launches = 0, threads = 0, guard_returns = 0, native = 0;
};

// one generated launch over a region with extents ex x ey and block bx x by
void count_launch(Stats& st, int64_t ex, int64_t ey, int64_t bx = 32, int64_t by = 4) {
  // cugridSize = ceiling(real(extent) / real(B)); non-positive grids are rejected
  auto ceil_div = [](int64_t e, int64_t b) -> int64_t {
    double q = static_cast<double>(e) / static_cast<double>(b);
    return static_cast<int64_t>(std::ceil(q));
  };
  int64_t gx = ceil_div(ex, bx), gy = ceil_div(ey, by);
  if (gx < 1 || gy < 1)
    fail(HFB_RUNTIME, "launch configuration dimensions must be positive");  // interp.cpp:1425
  int64_t total = gx * bx * gy * by;
  st.launches += 1;
  st.threads += total;
  st.guard_returns += total - ex * ey;
}

Span full_span(hfb_ctx* c, int64_t ni, int64_t nj) {
  Span sp;
  sp.ilo = 1;
  sp.ihi = ni;
  sp.jlo = 1;
  sp.jhi = nj;
  if (c->decomposed) {
    sp.i0 = c->decomp.i0;
    sp.j0 = c->decomp.j0;
    sp.gnx = c->decomp.global_nx;
    sp.gny = c->decomp.global_ny;
  } else {
    sp.gnx = ni;
    sp.gny = nj;
  }
  return sp;
}

Grid3 grid_of(const Slot& s) { return Grid3{s.lay.pitch, s.lay.plane}; }

cudaEvent_t take_event(hfb_ctx* c) {
  if (!c->free_events.empty()) {
    cudaEvent_t e = c->free_events.back();
    c->free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  cuda_check(cudaEventCreate(&e), "cudaEventCreate");
  return e;
}

// Launch one native kernel (or a fixed group of `n`), with optional CUDA-event timing
// on the context stream (never during graph capture).
// the stream a step kernel is launched on (see hfb_ctx::run_stream)
cudaStream_t ks(hfb_ctx* c) { return c->run_stream ? c->run_stream : c->stream; }

template <class F>
void launch(hfb_ctx* c, Stats& st, const char* name, F&& f, int n = 1) {
  NvtxRange nr(name);
  const bool timed = c->prof && !c->capturing;
  cudaEvent_t a = nullptr, b = nullptr;
  if (timed) {
    a = take_event(c);
    cuda_check(cudaEventRecord(a, ks(c)), "cudaEventRecord");
  }
  cuda_check(f(), name);
  if (timed) {
    b = take_event(c);
    cuda_check(cudaEventRecord(b, ks(c)), "cudaEventRecord");
    c->pending.push_back({name, a, b});
  }
  st.native += n;
}

void resolve_timings(hfb_ctx* c) {
  for (auto& t : c->pending) {
    cuda_check(cudaEventSynchronize(t.b), "cudaEventSynchronize");
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, t.a, t.b), "cudaEventElapsedTime");
    auto& acc = c->kernel_ms[t.name];
    acc.first += ms;
    acc.second += 1;
    c->free_events.push_back(t.a);
    c->free_events.push_back(t.b);
  }
  c->pending.clear();
}

// one array to exchange: its name on every rank (a module array, or "asu:<name>" for the
// ASUCA scheme's exchanged scratch), which of its buffers, this rank's origin of that
// buffer and its layout
struct XField {
  std::string name;
  int buf = 0;
  double* origin = nullptr;
  Grid3 g{};
  int64_t nk = 1;  // K extent times the trailing dimension
};
XField xfield(hfb_ctx* c, const char* name, int buf) {
  Slot& sl = slot(c, name);
  return XField{name, buf, sl.d_buf(buf), grid_of(sl), sl.lay.nk * sl.lay.nl};
}
std::vector<XField> xfields(hfb_ctx* c, const std::vector<const char*>& names) {
  std::vector<XField> v;
  for (const char* n : names) v.push_back(xfield(c, n, slot(c, n).cur));
  return v;
}
void halo_exchange_x(hfb_ctx* c, const std::vector<XField>& fields, cudaStream_t st);
void halo_exchange(hfb_ctx* c, const std::vector<const char*>& fields, int width,
                   cudaStream_t s = nullptr);
RemoteHalo remote_halo(hfb_ctx* c, const std::vector<Slot*>& f4);
void peer_signal(hfb_ctx* c, cudaStream_t st);

// Decomposed stencil step with the halo exchange overlapped: the exchange of `fields` goes
// to the communication stream; the columns at least `r` (the stencil radius) cells inside
// the tile — they never read the halo ring — are launched at once on the compute stream;
// the four boundary strips follow once the halos landed. Every column is computed from
// the same inputs either way, so the split is bit-identical to one full-span launch.
// `run(span)` launches the step kernel over a span of the tile; `xchg(stream)` enqueues
// the exchange (module arrays by name, or the ASUCA scheme's explicit buffers).
template <class X, class F>
void overlap_run(hfb_ctx* c, X&& xchg, int r, int64_t nx, int64_t ny, bool odd_ilo, F&& run) {
  const Span full = full_span(c, nx, ny);
  const bool multi = c->decomposed && c->decomp.px * c->decomp.py > 1;
  if (!multi) {
    run(full, false);
    return;
  }
  // The strips are whole tiles where the tile is large enough (32 columns, 4 rows: the
  // step kernels' CTA tile, so a strip launch does not run mostly idle lanes through the
  // whole K march; the interior is then whole tiles too), else r cells wide.
  // odd_ilo: spans must start at odd i (the step kernels' TMA boxes begin 2 columns left
  // of a tile and must start 16-B aligned), so an r-wide east strip may be one column
  // wider and an even interior start falls back to the serial order
  constexpr int64_t kTileI = 32, kTileJ = 4;
  Span in = full;
  auto split = [&](int64_t n, int64_t t, int64_t& lo, int64_t& hi) {
    lo = std::max<int64_t>(r, t) + 1;
    hi = lo - 1 + (n - r - (lo - 1)) / t * t;  // whole tiles, >= r short of the far edge
    if (hi >= lo && n - r - (lo - 1) > 0) return true;
    lo = r + 1;
    hi = n - r;
    return false;
  };
  if (!split(nx, kTileI, in.ilo, in.ihi) && odd_ilo && (nx - r + 1) % 2 == 0) --in.ihi;
  split(ny, kTileJ, in.jlo, in.jhi);
  if (!c->overlap || c->capturing || (odd_ilo && in.ilo % 2 == 0) || in.ihi < in.ilo ||
      in.jhi < in.jlo) {
    xchg(c->stream);
    run(full, true);
    return;
  }
  if (!c->comm) {
    cuda_check(cudaStreamCreateWithFlags(&c->comm, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming), "cudaEventCreate");
  }
  cuda_check(cudaEventRecord(c->ev_ready, c->stream), "cudaEventRecord");
  cuda_check(cudaStreamWaitEvent(c->comm, c->ev_ready, 0), "cudaStreamWaitEvent");
  xchg(c->comm);
  run(in, false);
  // the boundary strips follow the halo wait on the communication stream, so they run
  // alongside the interior launch (disjoint output columns, read-only inputs) instead of
  // after it; the compute stream joins them before the step ends
  Span south = full, north = full, west = full, east = full;
  south.jhi = in.jlo - 1;
  north.jlo = in.jhi + 1;
  west.jlo = east.jlo = in.jlo;
  west.jhi = east.jhi = in.jhi;
  west.ihi = in.ilo - 1;
  east.ilo = in.ihi + 1;
  c->run_stream = c->comm;
  try {
    for (const Span& sp : {south, north, west, east}) run(sp, true);
  } catch (...) {
    // the communication stream may still hold the exchange (a spinning wait) and strips:
    // join it before the error propagates, so nothing it does outlives the buffers
    c->run_stream = nullptr;
    cudaEventRecord(c->ev_halo, c->comm);
    cudaStreamWaitEvent(c->stream, c->ev_halo, 0);
    throw;
  }
  c->run_stream = nullptr;
  cuda_check(cudaEventRecord(c->ev_halo, c->comm), "cudaEventRecord");
  cuda_check(cudaStreamWaitEvent(c->stream, c->ev_halo, 0), "cudaStreamWaitEvent");
}
template <class F>
void exchange_and_run(hfb_ctx* c, const std::vector<const char*>& fields, int r, int64_t nx,
                      int64_t ny, bool odd_ilo, F&& run) {
  overlap_run(c, [&](cudaStream_t s) { halo_exchange(c, fields, r, s); }, r, nx, ny, odd_ilo,
              std::forward<F>(run));
}

// ---------------------------------------------------------------------------
// app: diffusion (diffusion.h90)
// ---------------------------------------------------------------------------
void diffusion_step(hfb_ctx* c, Stats& st, bool write_t_new) {
  int64_t nx = ival(c, "nx"), ny = ival(c, "ny"), nz = ival(c, "nz");
  double coef = rval(c, "coef");
  dev_read(c, "t_old");
  dev_write(c, "t_new");
  init_read(c, "t_old");  // the stencil and the boundary copy read every element
  Slot& to = slot(c, "t_old");
  Slot& tn = slot(c, "t_new");
  ensure_device(c, to, true);
  // hfk0 (stencil into the alternate t_old buffer [+ t_new]) then hfk1 fused away
  exchange_and_run(c, {"t_old"}, 1, nx, ny, false, [&](const Span& sp, bool) {
    launch(c, st, "hfk0_diffuse_step", [&] {
      if (c->force_generic)
        return launch_diffusion(to.d(), to.d_alt(), write_t_new ? tn.d() : nullptr,
                                grid_of(to), nz, coef, sp, ks(c));
      return launch_diffusion_ring(to.d(), to.d_alt(), write_t_new ? tn.d() : nullptr,
                                   grid_of(to), nz, to.lay.nj, coef, sp, ks(c));
    });
  });
  to.cur = to.alt();
  count_launch(st, nx, ny);
  count_launch(st, nx, ny);
  dev_written(c, "t_new");
  dev_written(c, "t_old");
  init_written(c, "t_new");
  init_written(c, "t_old");
}

void diffusion_entry(hfb_ctx* c, const std::string& r, Stats& st) {
  if (r == "main" || r == "simulation_run") {
    int64_t nsteps = ival(c, "nsteps");
    for (const char* n : {"t_new", "t_old"}) do_copy_to_device(c, slot(c, n));
    for (int64_t s = 0; s < nsteps; ++s) diffusion_step(c, st, s == nsteps - 1);
    for (const char* n : {"t_new", "t_old"}) entry_copy_out(c, slot(c, n));
  } else if (r == "diffuse_step") {
    diffusion_step(c, st, true);
  } else {
    fail(HFB_CONFIG, "program 'diffusion' has no entry '%s'", r.c_str());
  }
}

// ---------------------------------------------------------------------------
// app: damping (damping.h90)
// ---------------------------------------------------------------------------
void damping_kernel(hfb_ctx* c, Stats& st) {
  int64_t nx = ival(c, "nx_mx") - ival(c, "nx_mn") + 1;
  int64_t ny = ival(c, "ny_mx") - ival(c, "ny_mn") + 1;
  int64_t nz = ival(c, "nz_mx") - ival(c, "nz_mn") + 1;
  double t = rval(c, "tratio_bnd"), m = rval(c, "mtratio_bnd");
  count_launch(st, nx, ny);
  dev_read(c, "dens_ref_f");
  dev_read(c, "dens_ptb_bnd");
  dev_write(c, "dens_ptb_damp");
  init_read(c, "dens_ref_f");
  init_read(c, "dens_ptb_bnd");
  Slot& ref = slot(c, "dens_ref_f");
  Slot& bnd = slot(c, "dens_ptb_bnd");
  Slot& dmp = slot(c, "dens_ptb_damp");
  Span sp = full_span(c, nx, ny);
  launch(c, st, "hfk0_lateral_and_upper_damping", [&] { return launch_damping(ref.d(), bnd.d(), bnd.d() + bnd.lay.volume, dmp.d(), grid_of(ref), nz,
                          m, t, sp, c->stream); });
  dev_written(c, "dens_ptb_damp");
  init_written(c, "dens_ptb_damp");
}

void damping_entry(hfb_ctx* c, const std::string& r, Stats& st) {
  const char* names[] = {"dens_ptb_bnd", "dens_ptb_damp", "dens_ref_f"};
  if (r == "main") {
    for (const char* n : names) do_copy_to_device(c, slot(c, n));
    damping_kernel(c, st);
    for (const char* n : names) entry_copy_out(c, slot(c, n));
  } else if (r == "lateral_and_upper_damping") {
    damping_kernel(c, st);
  } else {
    fail(HFB_CONFIG, "program 'damping' has no entry '%s'", r.c_str());
  }
}

// ---------------------------------------------------------------------------
// app: bounded (bounded.h90)
// ---------------------------------------------------------------------------
void bounded_kernel(hfb_ctx* c, Stats& st) {
  int64_t nx = ival(c, "nx"), ny = ival(c, "ny");
  count_launch(st, (nx - 1) - 2 + 1, (ny - 1) - 2 + 1);
  dev_read(c, "a");
  dev_write(c, "b");
  Slot& a = slot(c, "a");
  Slot& b = slot(c, "b");
  if (a.dinit && nx >= 3 && ny >= 3) {  // 5-point interior update: all but the corners of a
    const int64_t lo1[2] = {1, 2}, hi1[2] = {nx, ny - 1}, lo2[2] = {2, 1}, hi2[2] = {nx - 1, ny};
    init_read(c, "a", lo1, hi1);
    init_read(c, "a", lo2, hi2);
  }
  halo_exchange(c, {"a"}, 1);
  Span sp = full_span(c, nx, ny);
  // startAt(2,2), endAt(nx-1, ny-1) on the GLOBAL domain
  sp.ilo = std::max<int64_t>(1, 2 - sp.i0);
  sp.ihi = std::min<int64_t>(nx, sp.gnx - 1 - sp.i0);
  sp.jlo = std::max<int64_t>(1, 2 - sp.j0);
  sp.jhi = std::min<int64_t>(ny, sp.gny - 1 - sp.j0);
  launch(c, st, "hfk0_interior_update", [&] { return launch_bounded(a.d(), b.d(), a.lay.pitch, sp, c->stream); });
  dev_written(c, "b");
  if (nx >= 3 && ny >= 3) {
    const int64_t lo[2] = {2, 2}, hi[2] = {nx - 1, ny - 1};
    init_written(c, "b", lo, hi);
  }
}

void bounded_entry(hfb_ctx* c, const std::string& r, Stats& st) {
  if (r == "main" || r == "simulation_run") {
    for (const char* n : {"a", "b"}) do_copy_to_device(c, slot(c, n));
    bounded_kernel(c, st);
    for (const char* n : {"a", "b"}) entry_copy_out(c, slot(c, n));
  } else if (r == "interior_update") {
    bounded_kernel(c, st);
  } else {
    fail(HFB_CONFIG, "program 'bounded' has no entry '%s'", r.c_str());
  }
}

// ---------------------------------------------------------------------------
// app: surface_flux (sf_state.h90, surface_flux.h90, driver.h90)
// ---------------------------------------------------------------------------
void sf_tile_kernel(hfb_ctx* c, Stats& st) {
  int64_t nx = ival(c, "nx"), ny = ival(c, "ny"), lt = ival(c, "tile_land");
  int64_t ntlm = ival(c, "ntlm");
  count_launch(st, nx, ny);
  dev_read(c, "cover_frac");
  for (const char* n : {"flx_sum_x", "flx_sum_y", "wind_speed"}) dev_write(c, n);
  if (lt < 1 || lt > ntlm)
    fail(HFB_RUNTIME, "index %lld out of bounds [1, %lld] in dimension 1 of 'cover_frac'",
         (long long)lt, (long long)ntlm);
  Slot& cf = slot(c, "cover_frac");
  {
    const int64_t lo[3] = {lt, 1, 1}, hi[3] = {lt, nx, ny};
    init_read(c, "cover_frac", lo, hi);
  }
  Span sp = full_span(c, nx, ny);
  launch(c, st, "hfk0_sf_slab_flx_tile_run", [&] { return launch_sf_tile(cf.d() + (lt - 1) * cf.lay.plane, slot(c, "flx_sum_x").d(),
                          slot(c, "flx_sum_y").d(), slot(c, "wind_speed").d(), cf.lay.pitch, sp,
                          c->stream); });
  for (const char* n : {"flx_sum_x", "flx_sum_y", "wind_speed"}) {
    dev_written(c, n);
    init_written(c, n);
  }
}

void sf_entry(hfb_ctx* c, const std::string& r, Stats& st) {
  const char* names[] = {"cover_frac", "flx_sum_x", "flx_sum_y", "wind_speed"};
  if (r == "main" || r == "simulation_run") {
    for (const char* n : names) do_copy_to_device(c, slot(c, n));
    if (r == "main") {
      // driver.h90 setup(): the host-side coverage shift, executed on the device copy
      // right after it arrives (same final state; no host compute on the product path)
      Slot& cf = slot(c, "cover_frac");
      int64_t nx = ival(c, "nx"), ny = ival(c, "ny");
      init_read(c, "cover_frac");
      launch(c, st, "sf_setup", [&] { return launch_sf_setup(cf.d(), grid_of(cf), ival(c, "ntlm"), full_span(c, nx, ny),
                               c->stream); });
      dev_written(c, "cover_frac");
    }
    sf_tile_kernel(c, st);
    for (const char* n : names) entry_copy_out(c, slot(c, n));
  } else if (r == "physics_run" || r == "sf_slab_flx_tile_run" || r == "physics_main") {
    sf_tile_kernel(c, st);
  } else {
    fail(HFB_CONFIG, "program 'surface_flux' has no device entry '%s'", r.c_str());
  }
}

// ---------------------------------------------------------------------------
// app: reduction (reduction.h90) — OpenACC-style reduction kernel
// ---------------------------------------------------------------------------
void allreduce_sum(hfb_ctx* c, double* dev_value);
const double* peer_gather(hfb_ctx* c, int64_t nx, int64_t ny);

void reduction_kernel(hfb_ctx* c, Stats& st) {
  int64_t nx = ival(c, "nx"), ny = ival(c, "ny"), nz = ival(c, "nz");
  double total = rval(c, "total");
  dev_read(c, "y");
  init_read(c, "y");
  Slot& y = slot(c, "y");
  if (!c->red_partials) {
    cuda_check(cudaMalloc(&c->red_partials, sizeof(double) * (reduce_partials_needed() + 2)),
               "cudaMalloc(partials)");
    c->red_result = c->red_partials + reduce_partials_needed();
    cuda_check(cudaMallocHost(&c->red_host, sizeof(double)), "cudaMallocHost");
  }
  Span sp = full_span(c, nx, ny);
  bool multi = c->decomposed && c->decomp.px * c->decomp.py > 1;
  bool local_group = multi && c->group != nullptr;
  if (c->reduce_ordered) {
    // the acc-simulated order (interp.cpp:1080-1173): column partials, then one in-order
    // pass from the initial value; a group assembles the tiles' partials in global order
    if (multi && !local_group && !c->peer)
      fail(HFB_CONFIG, "ordered reductions run single-domain, in an in-process group or over "
                       "the peer transport");
    const size_t need = static_cast<size_t>(nx) * static_cast<size_t>(ny);
    if (c->red_cols_cap < need) {
      if (c->red_cols) cudaFree(c->red_cols);
      c->red_cols = nullptr;
      cuda_check(cudaMalloc(&c->red_cols, need * sizeof(double)), "cudaMalloc(column sums)");
      c->red_cols_cap = need;
    }
    launch(c, st, "grid_total", [&] {
      return launch_column_sums(y.d(), grid_of(y), nz, sp, c->red_cols, nx, c->stream);
    });
    if (local_group) {  // combined in global (j, i) order by hfb_group_run
      st.launches += 1;
      st.threads += nx * ny;
      return;
    }
    // over the peer transport every rank gathers all tiles' partials in global order
    const double* cols = multi ? peer_gather(c, nx, ny) : c->red_cols;
    const int64_t count = multi ? c->decomp.global_nx * c->decomp.global_ny
                                : static_cast<int64_t>(need);
    launch(c, st, "grid_total_ordered", [&] {
      return launch_ordered_total(cols, count, total, c->red_result, c->stream);
    });
  } else {
    launch(c, st, "grid_total", [&] { return launch_grid_sum(y.d(), grid_of(y), nz, sp, c->red_partials, c->red_result,
                             multi ? 0.0 : total, c->stream); }, 2);
  }
  if (multi && !local_group && !c->reduce_ordered) allreduce_sum(c, c->red_result);
  cuda_check(cudaMemcpyAsync(c->red_host, c->red_result, sizeof(double), cudaMemcpyDeviceToHost,
                             c->stream),
             "cudaMemcpyAsync(total)");
  cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  Scalar& tot = c->scalars["total"];
  if (local_group) {
    c->red_local = *c->red_host;  // combined in rank order by hfb_group_run
  } else {
    tot.r = multi && !c->reduce_ordered ? total + *c->red_host : *c->red_host;
    tot.init = true;
  }
  // acc kernels: one virtual launch over the (j, i) iteration space (interp.cpp:1080-1114)
  st.launches += 1;
  st.threads += nx * ny;
}

void reduction_entry(hfb_ctx* c, const std::string& r, Stats& st) {
  if (r == "main" || r == "simulation_run") {
    do_copy_to_device(c, slot(c, "y"));
    Scalar& tot = c->scalars["total"];
    tot.r = 0.0;  // reduction.h90:34 `total = 0.0_r_size`
    tot.init = true;
    reduction_kernel(c, st);
    entry_copy_out(c, slot(c, "y"));
  } else if (r == "grid_total") {
    reduction_kernel(c, st);
  } else {
    fail(HFB_CONFIG, "program 'reduction' has no entry '%s'", r.c_str());
  }
}

// ---------------------------------------------------------------------------
// app: dycore (apps/dycore/dycore.h90)
// ---------------------------------------------------------------------------
PhysArgs phys_args(hfb_ctx* c, Slot& tsfc, Slot& colm) {
  const double dt = rval(c, "dt");
  return PhysArgs{tsfc.d(), colm.d(), dt * rval(c, "rrelax"), dt * rval(c, "ch")};
}

// column_physics on the current state (standalone kernel)
void column_physics(hfb_ctx* c, Stats& st) {
  int64_t nx = ival(c, "nx"), ny = ival(c, "ny"), nz = ival(c, "nz");
  for (const char* n : {"rho", "th", "u", "v", "tsfc", "colm"}) dev_read(c, n);
  for (const char* n : {"rho", "th", "tsfc", "colm"}) init_read(c, n);
  if (slot(c, "u").dinit) {  // the surface wind: u, v of the lowest level only
    const int64_t lo[3] = {1, 1, 1}, hi[3] = {1, nx, ny};
    init_read(c, "u", lo, hi);
    init_read(c, "v", lo, hi);
  }
  DynConst k = make_dyn_const(rval(c, "dt"), rval(c, "rdx"), rval(c, "rdy"), rval(c, "rdz"),
                              rval(c, "cs2"), rval(c, "grav"), rval(c, "th0"));
  Slot &rho = slot(c, "rho"), &th = slot(c, "th"), &u = slot(c, "u"), &v = slot(c, "v");
  PhysArgs ph = phys_args(c, slot(c, "tsfc"), slot(c, "colm"));
  launch(c, st, "column_physics", [&] {
    return launch_column_physics(rho.d(), th.d(), u.d(), v.d(), grid_of(th), nz, k, ph,
                                 full_span(c, nx, ny), c->stream);
  });
  count_launch(st, nx, ny);
  for (const char* n : {"th", "colm"}) {
    dev_written(c, n);
    init_written(c, n);
  }
}

// what a dynamics step reads of the prognostic state (every element except the C-grid
// wall planes u(nx), v(ny), w(nz), which the dialect never reads) and what it writes
void dyn_init_reads(hfb_ctx* c, bool with_physics) {
  for (const char* n : {"rho", "th", "p"}) init_read(c, n);
  init_read_but_last(c, "u", 1);  // (nz, nx, ny): i
  init_read_but_last(c, "v", 2);  // j
  init_read_but_last(c, "w", 0);  // k
  if (with_physics)
    for (const char* n : {"tsfc", "colm"}) init_read(c, n);
}
void dyn_init_writes(hfb_ctx* c, std::initializer_list<const char*> names) {
  for (const char* n : names) init_written(c, n);
}

// the fused warp-specialised step: cp.async-fed (product) or its TMA twin (measured
// slower, hfb_dycore_tma.cu)
cudaError_t launch_step(hfb_ctx* c, const DynIn& in, const DynOut& out, Grid3 g, int64_t nz,
                        int64_t nj, const DynConst& k, const Span& sp, cudaStream_t s,
                        const PhysArgs* phys = nullptr, const DynIn* base = nullptr) {
#ifdef HFB_VARIANTS
  if (c->force_ws2)
    return launch_dycore_step_ws2(in, out, g, nz, nj, k, sp, s, phys, base, c->debug_skip);
  if (c->force_tma)
    return launch_dycore_step_tma(in, out, g, nz, nj, k, sp, s, phys, base, c->debug_skip);
  if (c->arith_fma)
    return launch_dycore_step_ws_fma(in, out, g, nz, nj, k, sp, s, phys, base, nullptr,
                                     c->debug_skip);
  return launch_dycore_step_ws(in, out, g, nz, nj, k, sp, s, phys, base, nullptr,
                               c->debug_skip);
#else
  if (c->arith_fma) return launch_dycore_step_ws_fma(in, out, g, nz, nj, k, sp, s, phys, base);
  return launch_dycore_step_ws(in, out, g, nz, nj, k, sp, s, phys, base);
#endif
}

void dycore_step(hfb_ctx* c, Stats& st, bool with_physics = false) {
  int64_t nx = ival(c, "nx"), ny = ival(c, "ny"), nz = ival(c, "nz");
  if (nz < 2) fail(HFB_RUNTIME, "dycore_step needs nz >= 2 (got %lld)", (long long)nz);
  if (c->decomposed && c->decomp.px * c->decomp.py > 1 && c->decomp.halo < 2)
    fail(HFB_CONFIG, "dycore_step needs a halo of 2 cells (limited advection), got %d",
         c->decomp.halo);
  DynConst k = make_dyn_const(rval(c, "dt"), rval(c, "rdx"), rval(c, "rdy"), rval(c, "rdz"),
                              rval(c, "cs2"), rval(c, "grav"), rval(c, "th0"));
  for (const char* n : {"th", "u", "v", "w", "p", "rho"}) dev_read(c, n);
  if (with_physics)
    for (const char* n : {"tsfc", "colm"}) dev_read(c, n);
  dyn_init_reads(c, with_physics);
  Slot &rho = slot(c, "rho"), &th = slot(c, "th"), &u = slot(c, "u"), &v = slot(c, "v"),
       &w = slot(c, "w"), &p = slot(c, "p");
  for (Slot* s : {&th, &u, &v, &w, &p}) ensure_device(c, *s, true);
  DynIn in{rho.d(), th.d(), u.d(), v.d(), w.d(), p.d()};
  DynOut out{th.d_alt(), u.d_alt(), v.d_alt(), w.d_alt(), p.d_alt()};
  // the product kernel takes nz - 1 <= 128; the A/B variants (single role, TMA twin, two
  // columns per thread) keep their 64-face TMEM budget
  const bool variant = c->force_single_role || c->force_tma || c->force_ws2;
  const bool fused = (variant ? dycore_step_tmem_fits(nz) : dycore_step_ws_fits(nz)) &&
                     !c->force_generic && !c->force_split;
  const bool fused_physics = fused && !c->force_single_role && with_physics;
  PhysArgs ph{};
  if (fused_physics) ph = phys_args(c, slot(c, "tsfc"), slot(c, "colm"));
  // peer transport: the boundary strips store their outputs straight into the
  // neighbours' halo rings (the next step's exchange rides on this step's epilogue)
  const bool remote_ok = c->peer && fused && !c->force_single_role && !c->force_tma &&
                         !c->force_ws2;
  RemoteHalo rh{};
  if (remote_ok) rh = remote_halo(c, {&th, &u, &v, &p});
  exchange_and_run(c, {"th", "u", "v", "p"}, kHalo, nx, ny, true, [&](const Span& sp, bool edge) {
    const RemoteHalo* rem = remote_ok && edge ? &rh : nullptr;
    if (fused) {
      if (c->force_single_role)
        launch(c, st, "dycore_step", [&] {
          return launch_dycore_step_tmem(in, out, grid_of(th), nz, th.lay.nj, k, sp, ks(c));
        });
      else if (fused_physics)
        launch(c, st, "full_step", [&] {
          return rem ? (c->arith_fma ? launch_dycore_step_ws_fma : launch_dycore_step_ws)(
                           in, out, grid_of(th), nz, th.lay.nj, k, sp, ks(c), &ph, nullptr, rem, 0)
                     : launch_step(c, in, out, grid_of(th), nz, th.lay.nj, k, sp, ks(c), &ph);
        });
      else
        launch(c, st, "dycore_step", [&] {
          return rem ? (c->arith_fma ? launch_dycore_step_ws_fma : launch_dycore_step_ws)(
                           in, out, grid_of(th), nz, th.lay.nj, k, sp, ks(c), nullptr, nullptr,
                           rem, 0)
                     : launch_step(c, in, out, grid_of(th), nz, th.lay.nj, k, sp, ks(c));
        });
    } else {
      launch(c, st, "dycore_advect", [&] {
        return launch_dycore_advect(in, out.th, grid_of(th), nz, k, sp, ks(c));
      });
      if (dycore_acoustic_tmem_fits(nz) && !c->force_generic)
        launch(c, st, "dycore_acoustic", [&] {
          return launch_dycore_acoustic_tmem(in, out, grid_of(th), nz, th.lay.nj, k, sp,
                                             ks(c));
        });
      else
        launch(c, st, "dycore_acoustic", [&] {
          return launch_dycore_acoustic(in, out, grid_of(th), nz, k, sp, ks(c));
        });
    }
  });
  if (c->peer && c->decomp.px * c->decomp.py > 1) {
    if (remote_ok) peer_signal(c, c->stream);  // after the whole step: see peer_exchange
    c->peer_fused = remote_ok;
  }
  for (Slot* s : {&th, &u, &v, &w, &p}) s->cur = s->alt();
  // the generated code's 8 launches (dycore.h90 regions; region 1 spans i = 0..nx,
  // region 2 spans j = 0..ny)
  count_launch(st, nx + 1, ny);
  count_launch(st, nx, ny + 1);
  for (int r = 0; r < 6; ++r) count_launch(st, nx, ny);
  for (const char* n : {"th", "u", "v", "w", "p"}) dev_written(c, n);
  dyn_init_writes(c, {"th", "u", "v", "w", "p"});
  if (with_physics) {
    if (fused_physics) {
      count_launch(st, nx, ny);  // the generated code's column_physics launch
      dev_written(c, "colm");
      init_written(c, "colm");
    } else {
      column_physics(c, st);
    }
  }
}

// dycore.h90 rk3_step: Wicker-Skamarock RK3 with three native stage launches.
// Buffers per prognostic field: base (the state at the start of the step, left intact),
// s1 and s2 (stage states); the new state ends in s1.
void rk3_step(hfb_ctx* c, Stats& st) {
  int64_t nx = ival(c, "nx"), ny = ival(c, "ny"), nz = ival(c, "nz");
  if (!dycore_step_ws_fits(nz))
    fail(HFB_CONFIG, "rk3_step is implemented for 2 <= nz <= 129 (got %lld)", (long long)nz);
  if (c->decomposed && c->decomp.px * c->decomp.py > 1 && c->decomp.halo < 2)
    fail(HFB_CONFIG, "rk3_step needs a halo of 2 cells, got %d", c->decomp.halo);
  if (c->group)  // stage states are overwritten within a step: needs true rank lockstep
    fail(HFB_CONFIG, "rk3_step runs decomposed with one process per rank (NCCL), not in "
                     "an in-process group");
  const double dt = rval(c, "dt");
  for (const char* n : {"th", "u", "v", "w", "p", "rho"}) dev_read(c, n);
  dyn_init_reads(c, false);
  Slot &rho = slot(c, "rho"), &th = slot(c, "th"), &u = slot(c, "u"), &v = slot(c, "v"),
       &w = slot(c, "w"), &p = slot(c, "p");
  Slot* prog[5] = {&th, &u, &v, &w, &p};
  for (Slot* s : prog) ensure_device(c, *s, true, 3);
  const int b = th.cur;
  for (Slot* s : prog)
    if (s->cur != b) fail(HFB_RUNTIME, "prognostic buffers out of step");
  const int s1 = (b + 1) % 3, s2 = (b + 2) % 3;
  auto state = [&](int buf) {
    return DynIn{rho.d(), th.d_buf(buf), u.d_buf(buf), v.d_buf(buf), w.d_buf(buf), p.d_buf(buf)};
  };
  auto outs = [&](int buf) {
    return DynOut{th.d_buf(buf), u.d_buf(buf), v.d_buf(buf), w.d_buf(buf), p.d_buf(buf)};
  };
  const DynIn base = state(b);
  const double dts[3] = {dt / 3.0, dt / 2.0, dt};  // dycore.h90 rk3_step `dtf`
  const int cur_of[3] = {b, s1, s2}, out_of[3] = {s1, s2, s1};
  // the generated code's launches: the base copy region, then 8 regions per stage
  count_launch(st, nx, ny);
  for (int g = 0; g < 3; ++g) {
    // halos of the stage state (the current buffers of this stage)
    for (Slot* s : prog) s->cur = cur_of[g];
    DynConst k = make_dyn_const(dts[g], rval(c, "rdx"), rval(c, "rdy"), rval(c, "rdz"),
                                rval(c, "cs2"), rval(c, "grav"), rval(c, "th0"));
    const DynIn in = state(cur_of[g]);
    const DynOut out = outs(out_of[g]);
    exchange_and_run(c, {"th", "u", "v", "p"}, kHalo, nx, ny, true, [&](const Span& sp, bool) {
      launch(c, st, "rk3_stage", [&] {
        return launch_step(c, in, out, grid_of(th), nz, th.lay.nj, k, sp, ks(c), nullptr,
                           g == 0 ? nullptr : &base);
      });
    });
    count_launch(st, nx + 1, ny);
    count_launch(st, nx, ny + 1);
    for (int r = 0; r < 6; ++r) count_launch(st, nx, ny);
  }
  for (Slot* s : prog) s->cur = s1;
  for (const char* n : {"th", "u", "v", "w", "p"}) dev_written(c, n);
  dyn_init_writes(c, {"th", "u", "v", "w", "p"});
}

// apps/dycore/asuca.h90 asuca_step: the ASUCA time scheme (hfb_asuca.cu). Buffers per
// field: u, v, w, p — the state at the start of the step (base, left intact: every RK3
// stage restarts its acoustic sub-steps from it) and two that the short steps ping-pong
// between; theta, rho — base and the stage state (the stage end writes thb + dtf*fth in
// place of the previous stage's). The dialect's copies are these pointer choices.
void asuca_prepare(hfb_ctx* c) {
  for (const char* n : {"u", "v", "w", "p"}) ensure_device(c, slot(c, n), true, 3);
  for (const char* n : {"th", "rho"}) ensure_device(c, slot(c, n), true, 2);
  const int64_t elems = slot(c, "th").lay.alloc_elems;
  if (c->asu_elems != elems) {
    if (c->asu_exported)
      fail(HFB_CONFIG, "asuca_step: the layout changed after hfb_peer_export mapped the "
           "scheme's scratch arrays");
    for (double*& q : c->asu) {
      if (q) cudaFree(q);
      q = nullptr;
    }
    c->asu_elems = 0;
  }
  for (double*& q : c->asu) {
    if (q) continue;
    const size_t bytes = static_cast<size_t>(elems) * sizeof(double);
    cuda_check(cudaMalloc(&q, bytes), "cudaMalloc(asuca scratch)");
    cuda_check(cudaMemsetAsync(q, 0, bytes, c->stream), "cudaMemsetAsync");
  }
  c->asu_elems = elems;
}

void asuca_step(hfb_ctx* c, Stats& st) {
  const int64_t nx = ival(c, "nx"), ny = ival(c, "ny"), nz = ival(c, "nz");
  if (!asuca_fits(nz))
    fail(HFB_CONFIG, "asuca_step is implemented for 2 <= nz <= 129 (got %lld)", (long long)nz);
  // decomposed: every pass's stencil inputs are exchanged (peer or NCCL transport; push +
  // signal + wait per exchange, 28 per step with nsound = 6) on the communication stream
  // while the pass runs over the columns >= 2 cells inside the tile; the boundary strips
  // follow the halo wait (overlap_run; serial under graph capture or overlap=0)
  const bool multi = c->decomposed && c->decomp.px * c->decomp.py > 1;
  if (multi) {
    if (c->group)
      fail(HFB_CONFIG, "asuca_step on a decomposed context needs the peer or NCCL transport "
           "(in-process groups exchange module arrays only)");
    if (c->decomp.halo < 2)
      fail(HFB_CONFIG, "asuca_step needs a halo of 2 cells (decomposition halo %lld)",
           (long long)c->decomp.halo);
    if (c->peer && !c->asu_exported)
      fail(HFB_CONFIG, "asuca_step with the peer transport: set nsound before "
           "hfb_peer_export so the scheme's exchanged scratch arrays are mapped");
  }
  const int64_t nsound = ival(c, "nsound"), nbnd = ival(c, "nbnd"), kdmp = ival(c, "kdmp");
  const double dt = rval(c, "dt"), rdx = rval(c, "rdx"), rdy = rval(c, "rdy"),
               rdz = rval(c, "rdz"), cs2 = rval(c, "cs2"), grav = rval(c, "grav"),
               th0 = rval(c, "th0"), rdmp = rval(c, "rdmp"), rnbnd = rval(c, "rnbnd"),
               rnzd = rval(c, "rnzd");
  if (nsound < 1) fail(HFB_RUNTIME, "nsound must be >= 1 (got %lld)", (long long)nsound);
  for (const char* n : {"th", "u", "v", "w", "p", "rho"}) dev_read(c, n);
  dyn_init_reads(c, false);
  asuca_prepare(c);
  Slot &rho = slot(c, "rho"), &th = slot(c, "th"), &u = slot(c, "u"), &v = slot(c, "v"),
       &w = slot(c, "w"), &p = slot(c, "p");
  const int b = u.cur;
  for (Slot* s : {&v, &w, &p})
    if (s->cur != b) fail(HFB_RUNTIME, "prognostic buffers out of step");
  const int tb = th.cur, rb = rho.cur, tx = 1 - tb, rx = 1 - rb;
  const int x = (b + 1) % 3, y = (b + 2) % 3;
  const Grid3 g = grid_of(th);
  const int64_t nj = th.lay.nj;
  const Span sp = full_span(c, nx, ny);
  // the scratch fields share the prognostic fields' layout: views at their origin
  const int64_t o = th.lay.origin_off;
  double* const* A = c->asu;
  const AsuTend F{A[0] + o, A[1] + o, A[2] + o, A[3] + o, A[4] + o};
  double* pa = A[5] + o;
  const double dtau = dt / static_cast<double>(nsound);  // asuca.h90 `dt / real(nsound)`
  const AsuAcoConst ca = make_asu_aco_const(0.5 * dtau, dtau, rdx, rdy, rdz, cs2, grav, th0,
                                            rdmp, nbnd, kdmp, rnbnd, rnzd);
  const AsuAcoConst cb = make_asu_aco_const(dtau, dtau, rdx, rdy, rdz, cs2, grav, th0, rdmp,
                                            nbnd, kdmp, rnbnd, rnzd);
  count_launch(st, nx, ny);  // the base-state copy region
  const double* thS = th.d_buf(tb);
  const double* rhoS = rho.d_buf(rb);
  int us = b;  // buffer of the stage state's u, v, w (p's is unused by the tendencies)
  int ts = tb, rs = rb;  // buffers of the stage state's theta, rho
  // the exchanged scratch: every rank's origin of the same array (layout of th)
  auto xscratch = [&](const char* name, double* origin) {
    return XField{name, 0, origin, g, th.lay.nk * th.lay.nl};
  };
  if (multi) c->peer_fused = false;  // every exchange of the scheme is a push
  for (int stg = 1; stg <= 3; ++stg) {
    const double dtf = stg == 1 ? dt / 3.0 : stg == 2 ? dt / 2.0 : dt;
    const int64_t nsm = stg == 1 ? nsound / 3 : stg == 2 ? nsound / 2 : nsound;
    const AsuState S{rhoS, thS, u.d_buf(us), v.d_buf(us), w.d_buf(us), p.d_buf(us)};
    // the tendencies' stencils: the stage state with a 2-cell ring
    overlap_run(
        c,
        [&](cudaStream_t s) {
          halo_exchange_x(c, {xfield(c, "rho", rs), xfield(c, "th", ts), xfield(c, "u", us),
                              xfield(c, "v", us), xfield(c, "w", us)},
                          s);
        },
        2, nx, ny, true, [&](const Span& q, bool) {
          launch(c, st, "asuca_tend", [&] {
            return launch_asu_tend(S, F, g, nz, nj, rdx, rdy, rdz, q, ks(c));
          });
        });
    // the reference's launches: 12 flux regions (4 of them over an extra face row or
    // column), the theta/rho and the momentum tendencies, the acoustic restart copy
    count_launch(st, nx + 1, ny);
    count_launch(st, nx, ny + 1);
    count_launch(st, nx, ny);
    count_launch(st, nx, ny);
    count_launch(st, nx, ny + 1);
    count_launch(st, nx, ny);
    count_launch(st, nx + 1, ny);
    count_launch(st, nx, ny);
    count_launch(st, nx, ny);
    count_launch(st, nx + 1, ny);
    count_launch(st, nx, ny + 1);
    count_launch(st, nx, ny);
    count_launch(st, nx, ny);
    count_launch(st, nx, ny);
    count_launch(st, nx, ny);
    // the acoustic passes read fu(i-1), fv(j-1): exchanged with the first pass A
    bool fuv_pending = multi;
    int cur = b, nxt = x;
    for (int64_t ss = 0; ss < nsm; ++ss) {
      const AsuState C{rhoS, thS, u.d_buf(cur), v.d_buf(cur), w.d_buf(cur), p.d_buf(cur)};
      // pass A: p with its ring, u(i-1), v(j-1) of the short-step state
      overlap_run(
          c,
          [&](cudaStream_t s) {
            if (fuv_pending)
              halo_exchange_x(c, {xscratch("asu:fu", F.fu), xscratch("asu:fv", F.fv)}, s);
            halo_exchange_x(c, {xfield(c, "p", cur), xfield(c, "u", cur), xfield(c, "v", cur)},
                            s);
          },
          2, nx, ny, true, [&](const Span& q, bool) {
            launch(c, st, "asuca_acoustic_a", [&] {
              return launch_asu_acoustic(false, C, F.fu, F.fv, F.fw, nullptr, pa, nullptr,
                                         nullptr, nullptr, nullptr, g, nz, nj, ca, q, ks(c));
            });
          });
      fuv_pending = false;
      // pass B: pa's ring
      overlap_run(
          c, [&](cudaStream_t s) { halo_exchange_x(c, {xscratch("asu:pa", pa)}, s); }, 2, nx,
          ny, true, [&](const Span& q, bool) {
            launch(c, st, "asuca_acoustic_b", [&] {
              return launch_asu_acoustic(true, C, F.fu, F.fv, F.fw, pa, nullptr, u.d_buf(nxt),
                                         v.d_buf(nxt), w.d_buf(nxt), p.d_buf(nxt), g, nz, nj, cb,
                                         q, ks(c));
            });
          });
      for (int r = 0; r < 7; ++r) count_launch(st, nx, ny);
      cur = nxt;
      nxt = nxt == x ? y : x;
    }
    us = cur;
    launch(c, st, "asuca_stage_end", [&] {
      return launch_asu_stage_end(th.d_buf(tb), F.fth, rho.d_buf(rb), F.frho, th.d_buf(tx),
                                  rho.d_buf(rx), g, nz, dtf, sp, ks(c));
    });
    count_launch(st, nx, ny);
    thS = th.d_buf(tx);
    rhoS = rho.d_buf(rx);
    ts = tx;
    rs = rx;
  }
  for (Slot* s : {&u, &v, &w, &p}) s->cur = us;
  th.cur = tx;
  rho.cur = rx;
  for (const char* n : {"rho", "th", "u", "v", "w", "p"}) dev_written(c, n);
  dyn_init_writes(c, {"rho", "th", "u", "v", "w", "p"});
}

void dycore_entry(hfb_ctx* c, const std::string& r, Stats& st) {
  const char* names[] = {"p", "rho", "th", "u", "v", "w"};
  if (r == "main" || r == "simulation_run") {
    int64_t nsteps = ival(c, "nsteps");
    for (const char* n : names) do_copy_to_device(c, slot(c, n));
    for (int64_t s = 0; s < nsteps; ++s) dycore_step(c, st);
    for (const char* n : names) entry_copy_out(c, slot(c, n));
  } else if (r == "dycore_step") {
    dycore_step(c, st);
  } else if (r == "main_full" || r == "simulation_run_full") {
    int64_t nsteps = ival(c, "nsteps");
    const char* full_names[] = {"colm", "p", "rho", "th", "tsfc", "u", "v", "w"};
    for (const char* n : full_names) do_copy_to_device(c, slot(c, n));
    for (int64_t s = 0; s < nsteps; ++s) dycore_step(c, st, true);
    for (const char* n : full_names) entry_copy_out(c, slot(c, n));
  } else if (r == "full_step") {
    dycore_step(c, st, true);
  } else if (r == "rk3_step") {
    rk3_step(c, st);
  } else if (r == "main_rk3" || r == "simulation_run_rk3") {
    int64_t nsteps = ival(c, "nsteps");
    for (const char* n : names) do_copy_to_device(c, slot(c, n));
    for (int64_t s = 0; s < nsteps; ++s) rk3_step(c, st);
    for (const char* n : names) entry_copy_out(c, slot(c, n));
  } else if (r == "column_physics") {
    column_physics(c, st);
  } else if (r == "asuca_step") {
    asuca_step(c, st);
  } else if (r == "main_asuca" || r == "simulation_run_asuca") {
    int64_t nsteps = ival(c, "nsteps");
    for (const char* n : names) do_copy_to_device(c, slot(c, n));
    for (int64_t s = 0; s < nsteps; ++s) asuca_step(c, st);
    for (const char* n : names) entry_copy_out(c, slot(c, n));
  } else {
    fail(HFB_CONFIG, "program 'dycore' has no entry '%s'", r.c_str());
  }
}

using EntryFn = void (*)(hfb_ctx*, const std::string&, Stats&);
// a generated program: its host driver (hfb_plugin_desc::run) runs the routine
void plugin_entry(hfb_ctx* c, const std::string& r, Stats& st) {
  hfb_launch_stats s{};
  const int rc = c->app->plugin->run(c, r.c_str(), &s, 1);
  st.launches += s.launches;
  st.threads += s.threads;
  st.guard_returns += s.guard_returns;
  st.native += s.native_launches;
  if (rc == HFB_CONFIG && g_last_error.empty())
    fail(HFB_CONFIG, "program '%s' has no entry '%s'", c->app->app.c_str(), r.c_str());
  if (rc != HFB_OK) fail(rc, "%s", g_last_error.c_str());
}

EntryFn entry_fn(const AppDecl* d) {
  if (d->plugin) return plugin_entry;
  const std::string& app = d->app;
  if (app == "diffusion") return diffusion_entry;
  if (app == "damping") return damping_entry;
  if (app == "bounded") return bounded_entry;
  if (app == "surface_flux") return sf_entry;
  if (app == "reduction") return reduction_entry;
  if (app == "dycore") return dycore_entry;
  return nullptr;
}

bool entry_has_transfers(const AppDecl* d, const std::string& r) {
  if (d->plugin) {
    for (const char* const* e = d->plugin->transfer_entries; *e; ++e)
      if (r == *e) return true;
    return false;
  }
  const std::string& app = d->app;
  if (r == "main" || r == "simulation_run" || r == "main_full" || r == "simulation_run_full" ||
      r == "main_rk3" || r == "simulation_run_rk3" || r == "main_asuca" ||
      r == "simulation_run_asuca")
    return true;
  (void)app;
  return false;
}

std::string routine_name(const char* entry) {
  std::string r = lower(entry);
  if (r.rfind("hfd_", 0) == 0) r = r.substr(4);
  return r;
}

// ---------------------------------------------------------------------------
// multi-GPU: NCCL loaded lazily (only a decomposed context with >1 rank needs it)
// ---------------------------------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  int (*CommInitRank)(void**, int, const void* /*ncclUniqueId by value*/, int) = nullptr;
  int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

}  // namespace

// ncclUniqueId is a 128-byte struct passed by value; declare a matching type.
struct NcclId {
  char internal[128];
};
typedef int (*nccl_init_fn)(void**, int, NcclId, int);

namespace {

NcclApi& nccl() {
  static NcclApi api;
  if (!api.h) {
    api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!api.h) fail(HFB_CUDA, "cannot load libnccl.so.2: %s", dlerror());
    auto sym = [](const char* n) {
      void* p = dlsym(nccl().h, n);
      if (!p) fail(HFB_CUDA, "libnccl.so.2 lacks %s", n);
      return p;
    };
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.GetErrorString =
        reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  }
  return api;
}

void nccl_check(int rc, const char* what) {
  if (rc != 0) fail(HFB_CUDA, "%s: %s", what, nccl().GetErrorString(rc));
}

constexpr int kNcclFloat64 = 8;  // ncclDouble
constexpr int kNcclSum = 0;

// Two-phase halo update of `fields` (all share one layout): east/west faces first,
// then north/south faces spanning the I halo so corners arrive too.
void group_pull(hfb_ctx* c, const std::vector<const char*>& fields, cudaStream_t st);

// Peer-memory halo update: ONE push kernel stores this tile's boundary cells of every
// field into the halo rings of its (up to 8) neighbours — corners go straight to the
// diagonal neighbours, so there is a single phase —, a one-thread kernel releases the
// exchange epoch into each neighbour's flag, and a wait kernel acquires the flags of the
// neighbours that write into this tile. Everything is stream-ordered: the caller's
// stream sees the halos when the wait kernel retires. Lockstep is structural: a rank
// pushes exchange e only after its step e-1 (and so its reads of the halos exchange e-2
// wrote into the same buffers) has completed, and it cannot start step e before every
// neighbour's push e arrived.
// the neighbour directions of this tile (dx, dy, rank)
struct Nbr {
  int dx, dy, rank;
};
std::vector<Nbr> peer_neighbours(const hfb_decomp& d) {
  std::vector<Nbr> out;
  for (int dy = -1; dy <= 1; ++dy)
    for (int dx = -1; dx <= 1; ++dx) {
      if (dx == 0 && dy == 0) continue;
      const int rx = d.rx + dx, ry = d.ry + dy;
      if (rx < 0 || rx >= d.px || ry < 0 || ry >= d.py) continue;
      out.push_back({dx, dy, ry * d.px + rx});
    }
  return out;
}

void peer_wait(hfb_ctx* c, cudaStream_t st) {
  std::vector<const uint64_t*> mine;
  for (const Nbr& n : peer_neighbours(c->decomp))
    mine.push_back(c->peer_sig + kSigHalo + (n.dy + 1) * 3 + (n.dx + 1));
  cuda_check(launch_peer_wait(mine.data(), static_cast<int>(mine.size()),
                              c->peer_sig + kSigEpoch, st),
             "peer wait");
}

// release the next epoch to every neighbour (I am at offset (-dx, -dy) from each)
void peer_signal(hfb_ctx* c, cudaStream_t st) {
  ++c->halo_epoch;  // host mirror (statistics); the kernels use the device counter
  std::vector<uint64_t*> flags;
  for (const Nbr& n : peer_neighbours(c->decomp))
    flags.push_back(c->peers.at(n.rank).sig + kSigHalo + (1 - n.dy) * 3 + (1 - n.dx));
  cuda_check(launch_peer_signal(flags.data(), static_cast<int>(flags.size()),
                                c->peer_sig + kSigEpoch, st),
             "peer signal");
}

// where this tile's edge cells land in each neighbour's OUTPUT buffers (the buffer the
// current step writes: the neighbours flip their double buffers in lockstep)
RemoteHalo remote_halo(hfb_ctx* c, const std::vector<Slot*>& f4) {
  const hfb_decomp& d = c->decomp;
  RemoteHalo rh{};
  rh.nx = d.nx;
  rh.ny = d.ny;
  rh.h = d.halo;
  const char* names[4] = {"th", "u", "v", "p"};
  for (const Nbr& n : peer_neighbours(d)) {
    PeerRank& pr = c->peers.at(n.rank);
    const int q = rh.n++;
    rh.dx[q] = n.dx;
    rh.dy[q] = n.dy;
    rh.shift_i[q] = n.dx < 0 ? pr.nx : n.dx > 0 ? -d.nx : 0;
    rh.shift_j[q] = n.dy < 0 ? pr.ny : n.dy > 0 ? -d.ny : 0;
    double** dst[4] = {rh.th, rh.u, rh.v, rh.p};
    for (int fi = 0; fi < 4; ++fi) {
      const int b = f4[fi]->alt();
      auto it = pr.fields.find(names[fi]);
      if (it == pr.fields.end() || b >= it->second.nbuf || !it->second.base[b])
        fail(HFB_CONFIG, "peer transport: buffer %d of '%s' on rank %d is not mapped", b,
             names[fi], n.rank);
      const PeerField& rf = it->second;
      if (fi == 0) rh.g[q] = Grid3{rf.pitch, rf.plane};
      else if (rf.pitch != rh.g[q].pitch || rf.plane != rh.g[q].plane)
        fail(HFB_CONFIG, "peer transport: rank %d's fields differ in layout", n.rank);
      dst[fi][q] = rf.base[b] + rf.origin_off;
    }
  }
  return rh;
}

void peer_push_exchange(hfb_ctx* c, const std::vector<XField>& fields, cudaStream_t st);

void peer_exchange(hfb_ctx* c, const std::vector<const char*>& fields, cudaStream_t st) {
  NvtxRange nr("halo:peer");
  const hfb_decomp& d = c->decomp;
  const int64_t H = d.halo;
  if (H == 0) return;
  if (c->peer_fused) {  // the neighbours' previous step stored these halos already
    peer_wait(c, st);
    ++c->peer_handoffs;
    for (const Nbr& n : peer_neighbours(d))
      for (const char* f : fields) {
        Slot& sl = slot(c, f);
        c->halo_bytes += 2 * (n.dx == 0 ? d.nx : H) * (n.dy == 0 ? d.ny : H) * sl.lay.nk *
                         sl.lay.nl * static_cast<int64_t>(sizeof(double));
      }
    return;
  }
  peer_push_exchange(c, xfields(c, fields), st);
}

// one push + signal + wait exchange of the given buffers. Safe to reuse a buffer's halo
// ring at every exchange: a neighbour's last reads of that ring precede (in its stream
// order) its push of some exchange this rank waited for before pushing again
void peer_push_exchange(hfb_ctx* c, const std::vector<XField>& fields, cudaStream_t st) {
  const hfb_decomp& d = c->decomp;
  const int64_t H = d.halo;
  if (H == 0) return;
  ++c->halo_epoch;
  ++c->peer_pushes;
  PeerPush push{};
  std::vector<uint64_t*> remote_flags;
  std::vector<const uint64_t*> my_flags;
  for (int dy = -1; dy <= 1; ++dy)
    for (int dx = -1; dx <= 1; ++dx) {
      if (dx == 0 && dy == 0) continue;
      const int rx = d.rx + dx, ry = d.ry + dy;
      if (rx < 0 || rx >= d.px || ry < 0 || ry >= d.py) continue;
      const int nr = ry * d.px + rx;
      PeerRank& pr = c->peers.at(nr);
      // my boundary cells -> the neighbour's halo (its tile-local coordinates)
      const int64_t si0 = dx < 0 ? 1 : dx == 0 ? 1 : d.nx - H + 1;
      const int64_t nbi = dx == 0 ? d.nx : H;
      const int64_t di0 = dx < 0 ? pr.nx + 1 : dx == 0 ? 1 : 1 - H;
      const int64_t sj0 = dy < 0 ? 1 : dy == 0 ? 1 : d.ny - H + 1;
      const int64_t nbj = dy == 0 ? d.ny : H;
      const int64_t dj0 = dy < 0 ? pr.ny + 1 : dy == 0 ? 1 : 1 - H;
      for (const XField& f : fields) {
        auto it = pr.fields.find(f.name);
        if (it == pr.fields.end() || f.buf >= it->second.nbuf || !it->second.base[f.buf])
          fail(HFB_CONFIG, "peer transport: buffer %d of '%s' on rank %d is not mapped "
               "(export after binding every array)", f.buf, f.name.c_str(), nr);
        if (push.n == kMaxPeerBoxes) fail(HFB_CONFIG, "peer transport: too many halo boxes");
        const PeerField& rf = it->second;
        PeerBox& b = push.box[push.n++];
        b.src = f.origin;
        b.dst = rf.base[f.buf] + rf.origin_off;
        b.gs = f.g;
        b.gd = Grid3{rf.pitch, rf.plane};
        b.si0 = si0;
        b.sj0 = sj0;
        b.di0 = di0;
        b.dj0 = dj0;
        b.nbi = nbi;
        b.nbj = nbj;
        b.nk = f.nk;
        c->halo_bytes += 2 * nbi * nbj * b.nk * static_cast<int64_t>(sizeof(double));
      }
      // I am at offset (-dx, -dy) from the receiver
      remote_flags.push_back(pr.sig + kSigHalo + (1 - dy) * 3 + (1 - dx));
      my_flags.push_back(c->peer_sig + kSigHalo + (dy + 1) * 3 + (dx + 1));
    }
  cuda_check(launch_peer_push(push, st), "peer halo push");
  cuda_check(launch_peer_signal(remote_flags.data(), static_cast<int>(remote_flags.size()),
                                c->peer_sig + kSigEpoch, st),
             "peer signal");
  cuda_check(launch_peer_wait(my_flags.data(), static_cast<int>(my_flags.size()),
                              c->peer_sig + kSigEpoch, st),
             "peer wait");
}

void nccl_exchange(hfb_ctx* c, const std::vector<XField>& fields, cudaStream_t st);

void halo_exchange(hfb_ctx* c, const std::vector<const char*>& fields, int width,
                   cudaStream_t st) {
  if (!c->decomposed || c->decomp.px * c->decomp.py <= 1) return;
  if (!st) st = c->stream;
  if (c->peer) {
    peer_exchange(c, fields, st);
    return;
  }
  if (c->group) {
    group_pull(c, fields, st);
    return;
  }
  (void)width;  // the face boxes always carry the full halo ring (kHalo)
  nccl_exchange(c, xfields(c, fields), st);
}

// exchange of explicit buffers (peer or NCCL transport; in-process groups pull by name)
void halo_exchange_x(hfb_ctx* c, const std::vector<XField>& fields, cudaStream_t st) {
  if (!c->decomposed || c->decomp.px * c->decomp.py <= 1) return;
  if (c->peer) {
    NvtxRange nr("halo:peer");
    peer_push_exchange(c, fields, st);
    return;
  }
  if (c->group) fail(HFB_CONFIG, "in-process groups exchange module arrays only");
  nccl_exchange(c, fields, st);
}

// NCCL transport: two phases (west/east faces, then south/north spanning the I halo so
// the corners travel), all fields' boxes packed per side, grouped send/recv, unpack
void nccl_exchange(hfb_ctx* c, const std::vector<XField>& fields, cudaStream_t st) {
  if (!c->nccl_comm) fail(HFB_CONFIG, "decomposed context without a communicator");
  NvtxRange nr("halo:nccl");
  NcclApi& api = nccl();
  const hfb_decomp& d = c->decomp;
  const int nbr[4] = {d.west, d.east, d.south, d.north};
  for (int phase = 0; phase < 2; ++phase) {
    // per side: pack all fields' send boxes contiguously
    size_t need = 0;
    int64_t sbox[4][4], rbox[4][4];
    size_t count[4] = {0, 0, 0, 0};
    for (int s = 2 * phase; s < 2 * phase + 2; ++s) {
      hfb_decomp_faces(&d, s, sbox[s], rbox[s]);
      if (nbr[s] < 0) continue;
      for (const XField& f : fields)
        count[s] += static_cast<size_t>((sbox[s][1] - sbox[s][0] + 1) *
                                        (sbox[s][3] - sbox[s][2] + 1) * f.nk);
      need += count[s];
    }
    if (need == 0) continue;
    if (c->halo_cap < need) {
      if (c->halo_send) cudaFree(c->halo_send);
      if (c->halo_recv) cudaFree(c->halo_recv);
      cuda_check(cudaMalloc(&c->halo_send, need * sizeof(double)), "cudaMalloc(halo)");
      cuda_check(cudaMalloc(&c->halo_recv, need * sizeof(double)), "cudaMalloc(halo)");
      c->halo_cap = need;
    }
    size_t off = 0;
    size_t base[4] = {0, 0, 0, 0};
    for (int s = 2 * phase; s < 2 * phase + 2; ++s) {
      base[s] = off;
      if (nbr[s] < 0) continue;
      for (const XField& f : fields) {
        cuda_check(launch_pack_box(f.origin, c->halo_send + off, f.g, f.nk, sbox[s], true, st),
                   "halo pack");
        off += static_cast<size_t>((sbox[s][1] - sbox[s][0] + 1) * (sbox[s][3] - sbox[s][2] + 1) *
                                   f.nk);
      }
    }
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int s = 2 * phase; s < 2 * phase + 2; ++s) {
      if (nbr[s] < 0) continue;
      nccl_check(api.Send(c->halo_send + base[s], count[s], kNcclFloat64, nbr[s], c->nccl_comm,
                          st),
                 "ncclSend");
      nccl_check(api.Recv(c->halo_recv + base[s], count[s], kNcclFloat64, nbr[s], c->nccl_comm,
                          st),
                 "ncclRecv");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
    for (int s = 2 * phase; s < 2 * phase + 2; ++s) {
      if (nbr[s] < 0) continue;
      size_t o = base[s];
      for (const XField& f : fields) {
        cuda_check(launch_pack_box(f.origin, c->halo_recv + o, f.g, f.nk, rbox[s], false, st),
                   "halo unpack");
        o += static_cast<size_t>((rbox[s][1] - rbox[s][0] + 1) * (rbox[s][3] - rbox[s][2] + 1) *
                                 f.nk);
      }
      c->halo_bytes += static_cast<int64_t>(2 * count[s] * sizeof(double));
    }
  }
}

// In-process group: fill this rank's halo ring from the neighbours' interiors by device
// copies (pack into a staging buffer on this stream, unpack into the halo). A neighbour
// that already finished this step has flipped its double buffers; its previous state
// is then the other buffer (untouched until its next step).
void group_pull(hfb_ctx* c, const std::vector<const char*>& fields, cudaStream_t st) {
  const hfb_decomp& d = c->decomp;
  const int nbr[4] = {d.west, d.east, d.south, d.north};
  const int opposite[4] = {1, 0, 3, 2};
  for (int phase = 0; phase < 2; ++phase) {
    for (int s = 2 * phase; s < 2 * phase + 2; ++s) {
      if (nbr[s] < 0) continue;
      hfb_ctx* n = c->group->ranks[nbr[s]];
      int64_t my_send[4], my_recv[4], n_send[4], n_recv[4];
      hfb_decomp_faces(&d, s, my_send, my_recv);
      hfb_decomp_faces(&n->decomp, opposite[s], n_send, n_recv);
      for (const char* f : fields) {
        Slot& mine = slot(c, f);
        Slot& theirs = slot(n, f);
        if (!theirs.has_device) fail(HFB_RESIDENCY, "rank %d has no device copy of '%s'", nbr[s], f);
        const bool advanced = n->steps_done > c->steps_done;
        const double* src = (advanced && theirs.decl->pingpong && theirs.dev[1])
                                ? theirs.d_alt()
                                : theirs.d();
        const int64_t fk = mine.lay.nk * mine.lay.nl;
        const size_t cnt = static_cast<size_t>((n_send[1] - n_send[0] + 1) *
                                               (n_send[3] - n_send[2] + 1) * fk);
        if (cnt == 0) continue;
        if (c->halo_cap < cnt) {
          if (c->halo_send) cudaFree(c->halo_send);
          if (c->halo_recv) cudaFree(c->halo_recv);
          cuda_check(cudaMalloc(&c->halo_send, cnt * sizeof(double)), "cudaMalloc(halo)");
          cuda_check(cudaMalloc(&c->halo_recv, cnt * sizeof(double)), "cudaMalloc(halo)");
          c->halo_cap = cnt;
        }
        cuda_check(launch_pack_box(src, c->halo_send, grid_of(theirs), fk, n_send, true,
                                   st),
                   "group halo pack");
        cuda_check(launch_pack_box(mine.d(), c->halo_send, grid_of(mine), fk, my_recv, false,
                                   st),
                   "group halo unpack");
        c->halo_bytes += static_cast<int64_t>(cnt * sizeof(double));
      }
    }
    // the second phase reads the neighbours' I halos (corners): finish phase one everywhere
    cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  }
}

// ordered reductions over the peer transport: this tile's column partials are stored into
// every rank's gather buffer at their global (j, i) positions (parity of the reduction
// epoch), flags released; once every rank's flag arrived the buffer holds the whole
// plane in the acc-simulated combine order (linear id, i fastest)
const double* peer_gather(hfb_ctx* c, int64_t nx, int64_t ny) {
  const hfb_decomp& d = c->decomp;
  const int n = d.px * d.py;
  const int64_t G = d.global_nx * d.global_ny;
  const uint64_t epoch = ++c->red_epoch;
  const int64_t par = static_cast<int64_t>(epoch & 1) * G;
  if (n > 16) fail(HFB_CONFIG, "peer ordered reductions support up to 16 ranks");
  PeerPush push{};
  std::vector<uint64_t*> flags;
  std::vector<const uint64_t*> mine;
  for (int q = 0; q < n; ++q) {
    double* base = q == d.rank ? c->peer_gather : c->peers.at(q).gather;
    uint64_t* sig = q == d.rank ? c->peer_sig : c->peers.at(q).sig;
    PeerBox& b = push.box[push.n++];
    b.src = c->red_cols;
    b.dst = base + par;
    b.gs = Grid3{nx, 0};
    b.gd = Grid3{d.global_nx, 0};
    b.si0 = 1;
    b.sj0 = 1;
    b.di0 = d.i0 + 1;
    b.dj0 = d.j0 + 1;
    b.nbi = nx;
    b.nbj = ny;
    b.nk = 1;
    flags.push_back(sig + kSigRed + d.rank);
    mine.push_back(c->peer_sig + kSigRed + q);
  }
  cuda_check(launch_peer_push(push, c->stream), "peer gather push");
  cuda_check(launch_peer_signal(flags.data(), n, nullptr, c->stream, epoch), "peer signal");
  cuda_check(launch_peer_wait(mine.data(), n, nullptr, c->stream, epoch), "peer wait");
  return c->peer_gather + par;
}

void allreduce_sum(hfb_ctx* c, double* dev_value) {
  if (c->peer) {  // deterministic: every rank sums the partials in rank order
    const hfb_decomp& d = c->decomp;
    PeerReduce r{};
    r.value = dev_value;
    r.n = d.px * d.py;
    r.rank = d.rank;
    r.epoch = ++c->red_epoch;
    for (int q = 0; q < r.n; ++q) {
      uint64_t* base = q == d.rank ? c->peer_sig : c->peers.at(q).sig;
      r.slots[q] = reinterpret_cast<double*>(base + kSigSlots);
      r.flags[q] = base + kSigRed;
    }
    r.my_slots = reinterpret_cast<double*>(c->peer_sig + kSigSlots);
    r.my_flags = c->peer_sig + kSigRed;
    cuda_check(launch_peer_allreduce(r, c->stream), "peer all-reduce");
    return;
  }
  NcclApi& api = nccl();
  nccl_check(api.AllReduce(dev_value, dev_value, 1, kNcclFloat64, kNcclSum, c->nccl_comm,
                           c->stream),
             "ncclAllReduce");
}

}  // namespace

// ===========================================================================
// generated programs (include/hfb_plugin.h)
// ===========================================================================
namespace {

const AppDecl* load_plugin(const std::string& path) {
  static std::map<std::string, std::unique_ptr<AppDecl>> registry;
  auto it = registry.find(path);
  if (it != registry.end()) return it->second.get();
  void* h = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
  if (!h) fail(HFB_CONFIG, "cannot load program '%s': %s", path.c_str(), dlerror());
  auto get = reinterpret_cast<const hfb_plugin_desc* (*)()>(dlsym(h, "hfb_plugin"));
  if (!get) fail(HFB_CONFIG, "'%s' is not a program plugin (no hfb_plugin symbol)", path.c_str());
  const hfb_plugin_desc* d = get();
  if (!d || d->abi != HFB_PLUGIN_ABI)
    fail(HFB_CONFIG, "'%s': plugin ABI %d, expected %d", path.c_str(), d ? d->abi : -1,
         HFB_PLUGIN_ABI);
  auto decl = std::make_unique<AppDecl>();
  decl->app = lower(d->program);
  decl->module = lower(d->module);
  decl->plugin = d;
  for (const hfb_plugin_scalar* sc = d->scalars; sc->name; ++sc)
    decl->scalars.push_back({lower(sc->name), sc->type == 1 ? SType::Real : SType::Int});
  for (const hfb_plugin_array* ar = d->arrays; ar->name; ++ar) {
    ArrayDecl ad;
    ad.name = lower(ar->name);
    for (int q = 0; q < ar->rank; ++q) {
      ad.dims.push_back({ar->lower[q], ar->upper[q]});
      ad.roles.push_back(static_cast<Role>(ar->roles[q]));
    }
    decl->arrays.push_back(ad);
  }
  const AppDecl* out = decl.get();
  registry[path] = std::move(decl);
  return out;
}

bool is_scratch(const char* name) { return std::strchr(name, '.') != nullptr; }

void fill_view(const Layout& lay, const Role* roles, int rank, const int64_t* lower,
               double* origin, hfb_view* v) {
  v->origin = origin;
  for (int q = 0; q < 4; ++q) {
    v->stride[q] = 0;
    v->lower[q] = q < rank ? lower[q] : 1;
  }
  for (int q = 0; q < rank; ++q) {
    const Role r = roles[q];
    v->stride[q] = r == kRoleI ? 1 : r == kRoleJ ? lay.pitch : r == kRoleK ? lay.plane : lay.volume;
  }
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* hfb_last_error(void) { return g_last_error.c_str(); }
int hfb_abi_version(void) { return 2; }  // 2: state images, scenarios

hfb_status hfb_create(int device, hfb_ctx** out) {
  return guarded([&] {
    if (!out) fail(HFB_CONFIG, "null output pointer");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
      fail(HFB_CUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
    if (device < 0 || device >= n) fail(HFB_CONFIG, "device %d out of range [0, %d)", device, n);
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    auto c = std::make_unique<hfb_ctx>();
    c->device = device;
    cuda_check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    *out = c.release();
  });
}

void hfb_destroy(hfb_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->comm) cudaStreamSynchronize(c->comm);
  for (auto& [n, s] : c->slots) {
    for (double* p : s.dev)
      if (p) cudaFree(p);
    if (s.dinit) cudaFree(s.dinit);
    if (s.pinned && s.host) cudaHostUnregister(s.host);
    if (s.owned) cudaFreeHost(s.owned);
  }
  if (c->staging) cudaFree(c->staging);
  if (c->red_partials) cudaFree(c->red_partials);
  if (c->red_cols) cudaFree(c->red_cols);
  for (auto& kv : c->scratch) {
    if (kv.second.dev) cudaFree(kv.second.dev);
    if (kv.second.dinit) cudaFree(kv.second.dinit);
  }
  if (c->chk_flag) cudaFree(c->chk_flag);
  for (double* p : c->asu)
    if (p) cudaFree(p);
  if (c->red_host) cudaFreeHost(c->red_host);
  if (c->halo_send) cudaFree(c->halo_send);
  if (c->halo_recv) cudaFree(c->halo_recv);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  if (c->peer_sig) cudaFree(c->peer_sig);
  if (c->peer_gather) cudaFree(c->peer_gather);
  for (auto& kv : c->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  if (c->nccl_comm) nccl().CommDestroy(c->nccl_comm);
  for (auto& t : c->pending) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (cudaEvent_t e : c->free_events) cudaEventDestroy(e);
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  if (c->comm) cudaStreamDestroy(c->comm);
  cudaStreamDestroy(c->stream);
  delete c;
}

hfb_status hfb_load_program(hfb_ctx* c, const char* app) {
  return guarded([&] {
    if (!c) fail(HFB_CONFIG, "null context");
    std::string a = lower(app);
    const AppDecl* found = nullptr;
    const std::string path = app;
    if (path.size() > 3 && path.compare(path.size() - 3, 3, ".so") == 0)
      found = load_plugin(path);
    for (const AppDecl& d : app_table())
      if (d.app == a) found = &d;
    if (!found) fail(HFB_CONFIG, "unknown program '%s'", a.c_str());
    if (c->app) fail(HFB_CONFIG, "context already holds program '%s'", c->app->app.c_str());
    c->app = found;
    for (const ScalarDecl& s : found->scalars) {
      Scalar v;
      v.type = s.type;
      if (s.is_param) {
        v.i = static_cast<int64_t>(s.param);
        v.r = s.param;
        v.init = true;
      }
      c->scalars[s.name] = v;
    }
    for (const ArrayDecl& ad : found->arrays) {
      Slot s;
      s.module = found->module;
      s.name = ad.name;
      s.decl = &ad;
      s.stream = c->stream;
      c->slots[ad.name] = s;
    }
  });
}

hfb_status hfb_set_scalar_i64(hfb_ctx* c, const char* module, const char* name, int64_t v) {
  return guarded([&] {
    Scalar& s = scalar_ref(c, lower(module), lower(name));
    s.i = v;
    s.r = static_cast<double>(v);
    s.init = true;
  });
}

hfb_status hfb_set_scalar_f64(hfb_ctx* c, const char* module, const char* name, double v) {
  return guarded([&] {
    Scalar& s = scalar_ref(c, lower(module), lower(name));
    s.r = v;
    s.i = static_cast<int64_t>(v);
    s.init = true;
  });
}

hfb_status hfb_get_scalar_i64(hfb_ctx* c, const char* module, const char* name, int64_t* v) {
  return guarded([&] {
    Scalar& s = scalar_ref(c, lower(module), lower(name));
    if (!s.init) fail(HFB_RUNTIME, "read of unset variable '%s'", name);
    *v = s.type == SType::Int ? s.i : static_cast<int64_t>(s.r);
  });
}

hfb_status hfb_get_scalar_f64(hfb_ctx* c, const char* module, const char* name, double* v) {
  return guarded([&] {
    Scalar& s = scalar_ref(c, lower(module), lower(name));
    if (!s.init) fail(HFB_RUNTIME, "read of unset variable '%s'", name);
    *v = s.type == SType::Real ? s.r : static_cast<double>(s.i);
  });
}

hfb_status hfb_bind_init(hfb_ctx* c, const char* module, const char* name, uint8_t* init) {
  return guarded([&] {
    Slot& s = slot_ref(c, lower(module), lower(name));
    if (!s.host) fail(HFB_CONFIG, "bind the host buffer of '%s' before its init flags", name);
    s.hinit = init;
  });
}

hfb_status hfb_bind_array(hfb_ctx* c, const char* module, const char* name, int rank,
                          const int64_t* lo, const int64_t* hi, double* host,
                          const int64_t* strides, unsigned flags) {
  return guarded([&] {
    Slot& s = slot_ref(c, lower(module), lower(name));
    if (!host) fail(HFB_CONFIG, "null host buffer for '%s'", name);
    if (rank != static_cast<int>(s.decl->dims.size()))
      fail(HFB_RUNTIME, "array '%s' has rank %zu but is bound with rank %d", name,
           s.decl->dims.size(), rank);
    if (s.has_device || s.dev[0]) {
      // rebinding keeps the device buffers only if the shape is unchanged
      for (int d = 0; d < rank; ++d)
        if (lo[d] != s.lower[d] || hi[d] != s.upper[d])
          fail(HFB_CONFIG, "rebinding '%s' with a different shape after a transfer", name);
    }
    int64_t count = 1;
    int64_t ext[4];
    for (int d = 0; d < rank; ++d) {
      ext[d] = hi[d] - lo[d] + 1;
      if (ext[d] < 1) fail(HFB_RUNTIME, "non-positive extent for '%s'", name);
      count *= ext[d];
    }
    int64_t st[4];
    if (strides) {
      for (int d = 0; d < rank; ++d) st[d] = strides[d];
      // dense in some permutation: sorting dims by stride must give exact products
      int order[4] = {0, 1, 2, 3};
      std::sort(order, order + rank, [&](int a, int b) { return st[a] < st[b]; });
      int64_t expect = 1;
      for (int q = 0; q < rank; ++q) {
        int d = order[q];
        if (ext[d] > 1 && st[d] != expect)
          fail(HFB_CONFIG, "host buffer of '%s' is not dense (stride %lld, expected %lld)", name,
               (long long)st[d], (long long)expect);
        if (ext[d] == 1) st[d] = 0;
        expect *= ext[d];
      }
    } else {
      int64_t acc = 1;
      for (int d = rank - 1; d >= 0; --d) {  // ArrayValue order: last subscript fastest
        st[d] = ext[d] > 1 ? acc : 0;
        acc *= ext[d];
      }
    }
    if (s.pinned && s.host && s.host != host) {
      cudaHostUnregister(s.host);
      s.pinned = false;
    }
    if (s.owned && s.owned != host) {  // a caller buffer replaces a context-owned one
      cudaFreeHost(s.owned);
      s.owned = nullptr;
    }
    s.host = host;
    s.rank = rank;
    s.count = count;
    for (int d = 0; d < rank; ++d) {
      s.lower[d] = lo[d];
      s.upper[d] = hi[d];
      s.hstride[d] = st[d];
    }
    if ((flags & HFB_BIND_PIN) && !s.pinned) {
      cudaSetDevice(c->device);
      cudaError_t e = cudaHostRegister(host, static_cast<size_t>(count) * sizeof(double),
                                       cudaHostRegisterDefault);
      if (e == cudaSuccess)
        s.pinned = true;
      else
        cudaGetLastError();  // already pinned or not pinnable: transfers still work
    }
  });
}

hfb_status hfb_residency(hfb_ctx* c, const char* module, const char* name, int* residency,
                         int* has_device) {
  return guarded([&] {
    Slot& s = slot_ref(c, lower(module), lower(name));
    if (residency) *residency = s.res;
    if (has_device) *has_device = s.has_device ? 1 : 0;
  });
}

hfb_status hfrt_device_allocate(hfb_ctx* c, const char* module, const char* name) {
  return guarded([&] {
    cudaSetDevice(c->device);
    do_device_allocate(c, slot_ref(c, lower(module), lower(name)));
  });
}

hfb_status hfrt_copy_to_device(hfb_ctx* c, const char* module, const char* name) {
  return guarded([&] {
    cudaSetDevice(c->device);
    do_copy_to_device(c, slot_ref(c, lower(module), lower(name)));
  });
}

hfb_status hfrt_copy_from_device(hfb_ctx* c, const char* module, const char* name) {
  return guarded([&] {
    cudaSetDevice(c->device);
    do_copy_from_device(c, slot_ref(c, lower(module), lower(name)));
  });
}

hfb_status hfb_mark_host_modified(hfb_ctx* c, const char* module, const char* name) {
  return guarded([&] {
    Slot& s = slot_ref(c, lower(module), lower(name));
    if (s.has_device) s.res = kHost;
    c->peer_fused = false;
  });
}

static hfb_status run_impl(hfb_ctx* c, const char* entry, hfb_launch_stats* stats, bool sync,
                           bool allow_transfers) {
  return guarded([&] {
    if (!c || !c->app) fail(HFB_CONFIG, "no program loaded");
    cudaSetDevice(c->device);
    std::string r = routine_name(entry);
    if (!allow_transfers && entry_has_transfers(c->app, r))
      fail(HFB_CONFIG, "entry '%s' performs host transfers; use hfb_run", entry);
    NvtxRange nr(r.c_str());
    Stats st;
    // only consecutive dycore steps keep the fused halo hand-off; any other entry may
    // change the exchanged fields' buffers
    if (r != "dycore_step" && r != "full_step") c->peer_fused = false;
    entry_fn(c->app)(c, r, st);
    if (sync) cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    if (stats) {
      stats->launches = st.launches;
      stats->threads = st.threads;
      stats->guard_returns = st.guard_returns;
      stats->native_launches = st.native;
    }
  });
}

hfb_status hfb_run(hfb_ctx* c, const char* entry, hfb_launch_stats* stats) {
  return run_impl(c, entry, stats, true, true);
}

hfb_status hfb_enqueue(hfb_ctx* c, const char* entry, hfb_launch_stats* stats) {
  return run_impl(c, entry, stats, false, false);
}

hfb_status hfb_synchronize(hfb_ctx* c) {
  return guarded([&] { cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize"); });
}

void* hfb_stream(hfb_ctx* c) { return c ? c->stream : nullptr; }

// Capture `steps` calls of a stream-only entry into a CUDA graph (cached per entry, step
// count, starting buffer sides and peer hand-off state: a graph ending on the other
// buffer side is replayed from there by a second cached graph) and launch it.
void graph_launch(hfb_ctx* c, const char* entry, int64_t steps, hfb_launch_stats* stats,
                  bool sync) {
  if (!c || !c->app) fail(HFB_CONFIG, "no program loaded");
  if (steps < 1) return;
  cudaSetDevice(c->device);
  std::string r = routine_name(entry);
  if (entry_has_transfers(c->app, r))
    fail(HFB_CONFIG, "entry '%s' performs host transfers; cannot be graph-captured", entry);
  const bool multi = c->decomposed && c->decomp.px * c->decomp.py > 1;
  if (multi && !c->peer)
    fail(HFB_CONFIG, "graph replay of a decomposed context needs the peer transport "
         "(hfb_peer_attach); NCCL and in-process groups run the step loop");
  if (multi && c->app->app == "reduction")
    fail(HFB_CONFIG, "decomposed reductions gather through host-numbered epochs; run them "
         "with hfb_run");
  // no allocation may happen during capture: materialise every buffer first
  for (auto& [n, s] : c->slots)
    if (s.decl->pingpong && s.has_device) ensure_device(c, s, true, r == "rk3_step" ? 3 : 0);
  if (r == "asuca_step" && c->app->app == "dycore" && !c->app->plugin) asuca_prepare(c);
  std::string key = r + ":" + std::to_string(steps) + (c->peer_fused ? ":f" : ":p");
  for (auto& [n, s] : c->slots) key += ":" + n + "=" + std::to_string(s.cur);
  auto it = c->graphs.find(key);
  if (it == c->graphs.end()) {
    cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    std::map<std::string, int> cur0;
    for (auto& [n, s] : c->slots) cur0[n] = s.cur;
    const bool fused0 = c->peer_fused;
    const int64_t p0 = c->peer_pushes, h0 = c->peer_handoffs, b0 = c->halo_bytes,
                  e0 = static_cast<int64_t>(c->halo_epoch);
    Stats st;
    cudaGraph_t g;
    cuda_check(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal),
               "cudaStreamBeginCapture");
    c->capturing = true;
    try {
      for (int64_t s = 0; s < steps; ++s) entry_fn(c->app)(c, r, st);
      c->capturing = false;
    } catch (...) {
      c->capturing = false;
      cudaStreamEndCapture(c->stream, &g);
      for (auto& [n, s] : c->slots) s.cur = cur0[n];
      c->peer_fused = fused0;
      c->peer_pushes = p0;
      c->peer_handoffs = h0;
      c->halo_bytes = b0;
      c->halo_epoch = static_cast<uint64_t>(e0);
      throw;
    }
    cuda_check(cudaStreamEndCapture(c->stream, &g), "cudaStreamEndCapture");
    hfb_ctx::GraphEntry ge;
    cuda_check(cudaGraphInstantiate(&ge.exec, g, 0), "cudaGraphInstantiate");
    cudaGraphDestroy(g);
    for (auto& [n, s] : c->slots) ge.cur1[n] = s.cur;
    ge.stats = hfb_launch_stats{st.launches, st.threads, st.guard_returns, st.native};
    ge.peer_fused1 = c->peer_fused;
    ge.pushes = c->peer_pushes - p0;
    ge.handoffs = c->peer_handoffs - h0;
    ge.halo_bytes = c->halo_bytes - b0;
    ge.epochs = static_cast<int64_t>(c->halo_epoch) - e0;
    // capturing recorded the host-side effects without running anything: undo them, the
    // launch below applies them once
    for (auto& [n, s] : c->slots) s.cur = cur0[n];
    c->peer_fused = fused0;
    c->peer_pushes = p0;
    c->peer_handoffs = h0;
    c->halo_bytes = b0;
    c->halo_epoch = static_cast<uint64_t>(e0);
    it = c->graphs.emplace(key, std::move(ge)).first;
  }
  const hfb_ctx::GraphEntry& ge = it->second;
  cuda_check(cudaGraphLaunch(ge.exec, c->stream), "cudaGraphLaunch");
  for (auto& [n, sl] : c->slots) sl.cur = ge.cur1.at(n);
  c->peer_fused = ge.peer_fused1;
  c->peer_pushes += ge.pushes;
  c->peer_handoffs += ge.handoffs;
  c->halo_bytes += ge.halo_bytes;
  c->halo_epoch += static_cast<uint64_t>(ge.epochs);
  if (sync) cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  if (stats) *stats = ge.stats;
}

hfb_status hfb_run_graph(hfb_ctx* c, const char* entry, int64_t steps, hfb_launch_stats* stats) {
  return guarded([&] { graph_launch(c, entry, steps, stats, true); });
}

hfb_status hfb_enqueue_graph(hfb_ctx* c, const char* entry, int64_t steps,
                             hfb_launch_stats* stats) {
  return guarded([&] { graph_launch(c, entry, steps, stats, false); });
}

hfb_status hfb_device_array(hfb_ctx* c, const char* module, const char* name, hfb_array* out) {
  return guarded([&] {
    Slot& s = slot_ref(c, lower(module), lower(name));
    if (!s.has_device)
      fail(HFB_RESIDENCY, "array '%s' has no device copy (missing transfer)", name);
    hfb_array a{};
    a.origin = s.d();
    a.pitch = s.lay.pitch;
    a.plane = s.lay.plane;
    a.volume = s.lay.volume;
    a.rank = s.rank;
    for (int d = 0; d < 4; ++d) {
      a.lower[d] = s.lower[d];
      a.upper[d] = s.upper[d];
    }
    int packed = 0;
    for (int d = 0; d < s.rank; ++d) packed |= static_cast<int>(s.decl->roles[d]) << (2 * d);
    a.roles = packed;
    a.slot = &s;
    *out = a;
  });
}

// ---- generated-kernel ABI --------------------------------------------------
// The thread set of a launch: per axis (blockidx-1)*blockdim + threadidx (+start-1)
// for blockidx in 1..grid, threadidx in 1..block; guard `it > end` (codegen.cpp:495-512).
static Span launch_span(hfb_dim3 grid, hfb_dim3 block, int64_t istart, int64_t iend,
                        int64_t jstart, int64_t jend) {
  if (grid.x < 1 || grid.y < 1 || grid.z < 1 || block.x < 1 || block.y < 1 || block.z < 1)
    fail(HFB_RUNTIME, "launch configuration dimensions must be positive");
  Span sp;
  sp.ilo = istart;
  sp.jlo = jstart;
  sp.ihi = std::min<int64_t>(iend, istart - 1 + static_cast<int64_t>(grid.x) * block.x);
  sp.jhi = std::min<int64_t>(jend, jstart - 1 + static_cast<int64_t>(grid.y) * block.y);
  return sp;
}

static cudaStream_t stream_of(void* s, const hfb_array& a) {
  if (s) return static_cast<cudaStream_t>(s);
  return a.slot ? static_cast<const Slot*>(a.slot)->stream : nullptr;
}

hfb_status hfk0_diffuse_step(hfb_dim3 grid, hfb_dim3 block, double coef, int32_t k, int32_t nx,
                             int32_t ny, int32_t nz, hfb_array t_new, hfb_array t_old,
                             void* stream) {
  (void)k;
  return guarded([&] {
    Span sp = launch_span(grid, block, 1, nx, 1, ny);
    sp.gnx = nx;
    sp.gny = ny;
    cuda_check(launch_diffusion(t_old.origin, t_new.origin, nullptr,
                                Grid3{t_old.pitch, t_old.plane}, nz, coef, sp,
                                stream_of(stream, t_old)),
               "hfk0_diffuse_step");
  });
}

hfb_status hfk1_diffuse_step(hfb_dim3 grid, hfb_dim3 block, int32_t k, int32_t nx, int32_t ny,
                             int32_t nz, hfb_array t_new, hfb_array t_old, void* stream) {
  (void)k;
  return guarded([&] {
    Span sp = launch_span(grid, block, 1, nx, 1, ny);
    cuda_check(launch_copy_columns(t_new.origin, t_old.origin, Grid3{t_old.pitch, t_old.plane},
                                   nz, sp, stream_of(stream, t_old)),
               "hfk1_diffuse_step");
  });
}

hfb_status hfk0_lateral_and_upper_damping(hfb_dim3 grid, hfb_dim3 block, int32_t k,
                                          double mtratio_bnd, int32_t nx_mn, int32_t nx_mx,
                                          int32_t ny_mn, int32_t ny_mx, int32_t nz_mn,
                                          int32_t nz_mx, double tratio_bnd,
                                          hfb_array dens_ptb_bnd, hfb_array dens_ptb_damp,
                                          hfb_array dens_ref_f, void* stream) {
  (void)k;
  return guarded([&] {
    // i = (blockidx-1)*B + threadidx + nx_mn - 1, in array-relative 1-based terms
    Span sp = launch_span(grid, block, 1, nx_mx - nx_mn + 1, 1, ny_mx - ny_mn + 1);
    cuda_check(launch_damping(dens_ref_f.origin, dens_ptb_bnd.origin,
                              dens_ptb_bnd.origin + dens_ptb_bnd.volume, dens_ptb_damp.origin,
                              Grid3{dens_ref_f.pitch, dens_ref_f.plane}, nz_mx - nz_mn + 1,
                              mtratio_bnd, tratio_bnd, sp, stream_of(stream, dens_ref_f)),
               "hfk0_lateral_and_upper_damping");
  });
}

hfb_status hfk0_interior_update(hfb_dim3 grid, hfb_dim3 block, int32_t nx, int32_t ny,
                                hfb_array a, hfb_array b, void* stream) {
  return guarded([&] {
    Span sp = launch_span(grid, block, 2, nx - 1, 2, ny - 1);
    cuda_check(launch_bounded(a.origin, b.origin, a.pitch, sp, stream_of(stream, a)),
               "hfk0_interior_update");
  });
}

hfb_status hfk0_sf_slab_flx_tile_run(hfb_dim3 grid, hfb_dim3 block, int32_t nx, int32_t ny,
                                     int32_t tile_land, hfb_array cover_frac,
                                     hfb_array flx_sum_x, hfb_array flx_sum_y,
                                     hfb_array swind, void* stream) {
  return guarded([&] {
    Span sp = launch_span(grid, block, 1, nx, 1, ny);
    int64_t ntlm = cover_frac.upper[0] - cover_frac.lower[0] + 1;
    if (tile_land < 1 || tile_land > ntlm)
      fail(HFB_RUNTIME, "index %d out of bounds [1, %lld] in dimension 1 of 'cover_frac'",
           tile_land, (long long)ntlm);
    cuda_check(launch_sf_tile(cover_frac.origin + (tile_land - 1) * cover_frac.plane,
                              flx_sum_x.origin, flx_sum_y.origin, swind.origin, cover_frac.pitch,
                              sp, stream_of(stream, cover_frac)),
               "hfk0_sf_slab_flx_tile_run");
  });
}

// ---- decomposition -----------------------------------------------------------
hfb_status hfb_decomp_init(hfb_decomp* d) {
  return guarded([&] {
    if (!d) fail(HFB_CONFIG, "null decomposition");
    if (d->px < 1 || d->py < 1) fail(HFB_CONFIG, "process grid must be positive");
    if (d->rank < 0 || d->rank >= d->px * d->py) fail(HFB_CONFIG, "rank out of range");
    if (d->halo < 0 || d->halo > kHalo) fail(HFB_CONFIG, "halo width must be in [0, %d]", kHalo);
    if (d->global_nx < d->px || d->global_ny < d->py)
      fail(HFB_CONFIG, "grid %lldx%lld cannot be split %dx%d", (long long)d->global_nx,
           (long long)d->global_ny, d->px, d->py);
    d->rx = d->rank % d->px;
    d->ry = d->rank / d->px;
    auto split = [](int64_t n, int p, int r, int64_t* off, int64_t* len) {
      int64_t base = n / p, rem = n % p;
      *len = base + (r < rem ? 1 : 0);
      *off = r * base + std::min<int64_t>(r, rem);
    };
    split(d->global_nx, d->px, d->rx, &d->i0, &d->nx);
    split(d->global_ny, d->py, d->ry, &d->j0, &d->ny);
    if (d->halo > 0 && (d->nx < d->halo || d->ny < d->halo))
      fail(HFB_CONFIG, "tile %lldx%lld is narrower than the halo", (long long)d->nx,
           (long long)d->ny);
    d->west = d->rx > 0 ? d->rank - 1 : -1;
    d->east = d->rx < d->px - 1 ? d->rank + 1 : -1;
    d->south = d->ry > 0 ? d->rank - d->px : -1;
    d->north = d->ry < d->py - 1 ? d->rank + d->px : -1;
  });
}

hfb_status hfb_decomp_faces(const hfb_decomp* d, int32_t side, int64_t send_box[4],
                            int64_t recv_box[4]) {
  return guarded([&] {
    if (!d) fail(HFB_CONFIG, "null decomposition");
    const int64_t H = d->halo, nx = d->nx, ny = d->ny;
    int64_t sb[4], rb[4];
    switch (side) {
      case 0:  // west: send my first H columns, receive the H columns left of me
        sb[0] = 1; sb[1] = H; sb[2] = 1; sb[3] = ny;
        rb[0] = 1 - H; rb[1] = 0; rb[2] = 1; rb[3] = ny;
        break;
      case 1:  // east
        sb[0] = nx - H + 1; sb[1] = nx; sb[2] = 1; sb[3] = ny;
        rb[0] = nx + 1; rb[1] = nx + H; rb[2] = 1; rb[3] = ny;
        break;
      case 2:  // south, spanning the I halo (corners)
        sb[0] = 1 - H; sb[1] = nx + H; sb[2] = 1; sb[3] = H;
        rb[0] = 1 - H; rb[1] = nx + H; rb[2] = 1 - H; rb[3] = 0;
        break;
      case 3:  // north
        sb[0] = 1 - H; sb[1] = nx + H; sb[2] = ny - H + 1; sb[3] = ny;
        rb[0] = 1 - H; rb[1] = nx + H; rb[2] = ny + 1; rb[3] = ny + H;
        break;
      default:
        fail(HFB_CONFIG, "side must be 0..3");
    }
    const int nb[4] = {d->west, d->east, d->south, d->north};
    if (nb[side] < 0 || H == 0) {
      sb[1] = sb[0] - 1;
      rb[1] = rb[0] - 1;
    }
    for (int q = 0; q < 4; ++q) {
      send_box[q] = sb[q];
      recv_box[q] = rb[q];
    }
  });
}

hfb_status hfb_layout_of(int64_t ni, int64_t nj, int64_t nk, int64_t nl, int64_t* pitch,
                         int64_t* plane, int64_t* alloc_elems, int64_t* origin_off) {
  return guarded([&] {
    if (ni < 1 || nj < 1 || nk < 1 || nl < 1) fail(HFB_CONFIG, "non-positive extent");
    const Layout L = Layout::make(ni, nj, nk, nl);
    *pitch = L.pitch;
    *plane = L.plane;
    *alloc_elems = L.alloc_elems;
    *origin_off = L.origin_off;
  });
}

hfb_status hfb_pack_box_host(const double* origin, int64_t pitch, int64_t plane, int64_t nk,
                             const int64_t box[4], double* buf) {
  return guarded([&] { pack_box_host(origin, buf, Grid3{pitch, plane}, nk, box, true); });
}

hfb_status hfb_unpack_box_host(double* origin, int64_t pitch, int64_t plane, int64_t nk,
                               const int64_t box[4], const double* buf) {
  return guarded([&] {
    pack_box_host(origin, const_cast<double*>(buf), Grid3{pitch, plane}, nk, box, false);
  });
}

hfb_status hfb_set_decomposition(hfb_ctx* c, const hfb_decomp* d, const void* nccl_id) {
  return guarded([&] {
    if (!c) fail(HFB_CONFIG, "null context");
    hfb_decomp dd = *d;
    hfb_status st = hfb_decomp_init(&dd);
    if (st != HFB_OK) fail(st, "%s", g_last_error.c_str());
    c->decomp = dd;
    c->decomposed = true;
    if (dd.px * dd.py > 1 && nccl_id) {  // NULL: the rank joins an in-process group
      cudaSetDevice(c->device);
      NcclApi& api = nccl();
      (void)api;
      auto init = reinterpret_cast<nccl_init_fn>(dlsym(api.h, "ncclCommInitRank"));
      if (!init) fail(HFB_CUDA, "libnccl.so.2 lacks ncclCommInitRank");
      NcclId id;
      std::memcpy(id.internal, nccl_id, sizeof id.internal);
      nccl_check(init(&c->nccl_comm, dd.px * dd.py, id, dd.rank), "ncclCommInitRank");
    }
  });
}

int64_t hfb_halo_bytes(hfb_ctx* c) { return c ? c->halo_bytes : 0; }

hfb_status hfb_transfer_bytes(hfb_ctx* c, int64_t* h2d, int64_t* d2h) {
  return guarded([&] {
    if (!c) fail(HFB_CONFIG, "null context");
    if (h2d) *h2d = c->h2d_bytes;
    if (d2h) *d2h = c->d2h_bytes;
  });
}

hfb_status hfb_group_create(hfb_ctx* const* ctxs, int n, hfb_group** out) {
  return guarded([&] {
    if (!ctxs || n < 1 || !out) fail(HFB_CONFIG, "bad group arguments");
    auto g = std::make_unique<hfb_group>();
    for (int r = 0; r < n; ++r) {
      hfb_ctx* c = ctxs[r];
      if (!c || !c->app) fail(HFB_CONFIG, "rank %d has no program", r);
      if (!c->decomposed || c->decomp.rank != r || c->decomp.px * c->decomp.py != n)
        fail(HFB_CONFIG, "rank %d: decomposition rank/size does not match the group", r);
      if (c->app != ctxs[0]->app) fail(HFB_CONFIG, "ranks run different programs");
      if (c->group) fail(HFB_CONFIG, "rank %d already belongs to a group", r);
      g->ranks.push_back(c);
    }
    for (hfb_ctx* c : g->ranks) {
      c->group = g.get();
      c->steps_done = 0;
    }
    *out = g.release();
  });
}

void hfb_group_destroy(hfb_group* g) {
  if (!g) return;
  for (hfb_ctx* c : g->ranks) c->group = nullptr;
  delete g;
}

// Lockstep execution of one entry on every rank of an in-process group. Per-step
// entries run rank by rank (each pulls its halos first); `main`/`simulation_run` are
// unrolled into copy-in on all ranks, nsteps x (step on every rank), copy-out.
hfb_status hfb_group_run(hfb_group* g, const char* entry, hfb_launch_stats* stats) {
  return guarded([&] {
    if (!g || g->ranks.empty()) fail(HFB_CONFIG, "empty group");
    std::string r = routine_name(entry);
    const std::string& app = g->ranks[0]->app->app;
    Stats st;
    auto each = [&](const std::function<void(hfb_ctx*)>& f) {
      for (hfb_ctx* c : g->ranks) {
        cudaSetDevice(c->device);
        f(c);
        cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
      }
    };
    const bool full = r == "main_full" || r == "simulation_run_full";
    const bool outer = r == "main" || r == "simulation_run" || full;
    std::vector<std::string> transfers;
    std::string step;
    if (app == "dycore" && full) {
      transfers = {"colm", "p", "rho", "th", "tsfc", "u", "v", "w"};
      step = "full_step";
    } else if (app == "dycore") {
      transfers = {"p", "rho", "th", "u", "v", "w"};
      step = "dycore_step";
    } else if (app == "diffusion") {
      transfers = {"t_new", "t_old"};
      step = "diffuse_step";
    } else if (app == "bounded") {
      transfers = {"a", "b"};
      step = "interior_update";
    } else if (app == "damping") {
      transfers = {"dens_ptb_bnd", "dens_ptb_damp", "dens_ref_f"};
      step = "lateral_and_upper_damping";
    } else if (app == "surface_flux") {
      transfers = {"cover_frac", "flx_sum_x", "flx_sum_y", "wind_speed"};
      step = "physics_run";
    } else if (app == "reduction") {
      transfers = {"y"};
      step = "grid_total";
    }
    if (outer && app == "surface_flux" && r == "main")
      fail(HFB_CONFIG, "group runs of surface_flux start at simulation_run");
    if (!outer) step = r;
    int64_t nsteps = 1;
    if (outer && (app == "dycore" || app == "diffusion")) nsteps = ival(g->ranks[0], "nsteps");
    if (outer) each([&](hfb_ctx* c) {
      for (const std::string& n : transfers) do_copy_to_device(c, slot(c, n.c_str()));
      if (app == "reduction") {
        c->scalars["total"].r = 0.0;
        c->scalars["total"].init = true;
      }
    });
    double total0 = app == "reduction" ? rval(g->ranks[0], "total") : 0.0;
    for (int64_t s = 0; s < nsteps; ++s) {
      each([&](hfb_ctx* c) {
        Stats local;
        if (app == "diffusion" && step == "diffuse_step")
          diffusion_step(c, local, !outer || s == nsteps - 1);
        else
          entry_fn(g->ranks[0]->app)(c, step, local);
        if (c == g->ranks[0]) st = Stats{st.launches + local.launches, st.threads + local.threads,
                                         st.guard_returns + local.guard_returns,
                                         st.native + local.native};
        else
          st.native += local.native;
        c->steps_done += 1;  // later ranks of this step pull this rank's previous state
      });
    }
    if (app == "reduction" && g->ranks[0]->reduce_ordered) {
      // every rank's column partials into rank 0's global buffer in (j, i) order, then
      // the in-order pass from the initial value (interp.cpp:1163-1173)
      hfb_ctx* r0 = g->ranks[0];
      const hfb_decomp& d0 = r0->decomp;
      const size_t gcount = static_cast<size_t>(d0.global_nx) * static_cast<size_t>(d0.global_ny);
      double* gcols = nullptr;
      cudaSetDevice(r0->device);
      for (hfb_ctx* c : g->ranks) cuda_check(cudaStreamSynchronize(c->stream), "sync");
      cuda_check(cudaMalloc(&gcols, gcount * sizeof(double)), "cudaMalloc(global column sums)");
      struct Free { double* p; ~Free() { cudaFree(p); } } free_g{gcols};
      for (hfb_ctx* c : g->ranks)
        cuda_check(cudaMemcpy2DAsync(gcols + c->decomp.j0 * d0.global_nx + c->decomp.i0,
                                     d0.global_nx * sizeof(double), c->red_cols,
                                     c->decomp.nx * sizeof(double), c->decomp.nx * sizeof(double),
                                     c->decomp.ny, cudaMemcpyDefault, r0->stream),
                   "cudaMemcpy2DAsync(column sums)");
      cuda_check(launch_ordered_total(gcols, static_cast<int64_t>(gcount), total0, r0->red_result,
                                      r0->stream),
                 "ordered total");
      st.native += 1;
      cuda_check(cudaMemcpyAsync(r0->red_host, r0->red_result, sizeof(double),
                                 cudaMemcpyDeviceToHost, r0->stream),
                 "cudaMemcpyAsync(total)");
      cuda_check(cudaStreamSynchronize(r0->stream), "cudaStreamSynchronize");
      for (hfb_ctx* c : g->ranks) {
        c->scalars["total"].r = *r0->red_host;
        c->scalars["total"].init = true;
      }
    } else if (app == "reduction") {
      double sum = 0.0;
      for (hfb_ctx* c : g->ranks) sum += c->red_local;  // rank order: deterministic
      for (hfb_ctx* c : g->ranks) {
        c->scalars["total"].r = total0 + sum;
        c->scalars["total"].init = true;
      }
    }
    if (outer) each([&](hfb_ctx* c) {
      for (const std::string& n : transfers) do_copy_from_device(c, slot(c, n.c_str()));
    });
    if (stats) *stats = hfb_launch_stats{st.launches, st.threads, st.guard_returns, st.native};
  });
}

const char* hfb_program_module(hfb_ctx* c) {
  return c && c->app ? c->app->module.c_str() : nullptr;
}

const char* hfb_program_name(hfb_ctx* c) { return c && c->app ? c->app->app.c_str() : nullptr; }

hfb_status hfb_set_option(hfb_ctx* c, const char* key, const char* value) {
  return guarded([&] {
    if (!c) fail(HFB_CONFIG, "null context");
    const std::string k = key ? key : "", v = value ? value : "";
    if (k == "variant") {
      c->force_generic = v == "generic";
      c->force_split = v == "split";
      c->force_single_role = v == "single_role";
      c->force_tma = v == "tma";
      c->force_ws2 = v == "ws2";
      const bool known = v == "product" || v == "generic" || v == "split" ||
                         v == "single_role" || v == "tma" || v == "ws2";
      if (!known) {
        c->force_tma = c->force_ws2 = false;
        fail(HFB_CONFIG, "unknown kernel variant '%s' (product, generic, split, single_role, "
             "tma, ws2)", v.c_str());
      }
#ifndef HFB_VARIANTS
      if (c->force_tma || c->force_ws2) {
        c->force_tma = c->force_ws2 = false;
        fail(HFB_CONFIG, "kernel variant '%s' is not compiled into this library (A/B build: "
             "make -C csrc variants -> libhfb_variants.so)", v.c_str());
      }
#endif
    } else if (k == "checked") {
      if (v != "0" && v != "1") fail(HFB_CONFIG, "option checked takes 0 or 1, got '%s'", v.c_str());
      c->checked = v == "1";
    } else if (k == "arith") {
      if (v != "exact" && v != "fma")
        fail(HFB_CONFIG, "option arith takes exact or fma, got '%s'", v.c_str());
      c->arith_fma = v == "fma";
    } else if (k == "overlap") {
      if (v != "0" && v != "1") fail(HFB_CONFIG, "option overlap takes 0 or 1, got '%s'", v.c_str());
      c->overlap = v == "1";
    } else if (k == "debug_skip") {
#ifdef HFB_VARIANTS
      c->debug_skip = std::atoi(v.c_str());
#else
      fail(HFB_CONFIG, "option debug_skip exists only in the A/B build (libhfb_variants.so)");
#endif
    } else {
      fail(HFB_CONFIG, "unknown option '%s' (variant, arith, checked, overlap, debug_skip)",
           k.c_str());
    }
  });
}

int hfb_variants_build(void) {
#ifdef HFB_VARIANTS
  return 1;
#else
  return 0;
#endif
}

hfb_status hfb_set_reduction_order(hfb_ctx* c, int ordered) {
  return guarded([&] {
    if (!c) fail(HFB_CONFIG, "null context");
    c->reduce_ordered = ordered != 0;
  });
}

hfb_status hfb_profile(hfb_ctx* c, int enable) {
  return guarded([&] {
    if (!c) fail(HFB_CONFIG, "null context");
    resolve_timings(c);
    if (enable < 0) c->kernel_ms.clear();
    c->prof = enable > 0;
  });
}

hfb_status hfb_kernel_time(hfb_ctx* c, const char* kernel, double* total_ms, int64_t* count) {
  return guarded([&] {
    if (!c) fail(HFB_CONFIG, "null context");
    resolve_timings(c);
    auto it = c->kernel_ms.find(kernel ? kernel : "");
    *total_ms = it == c->kernel_ms.end() ? 0.0 : it->second.first;
    *count = it == c->kernel_ms.end() ? 0 : it->second.second;
  });
}

hfb_status hfb_nccl_unique_id(void* out128) {
  return guarded([&] {
    auto get = reinterpret_cast<int (*)(NcclId*)>(dlsym(nccl().h, "ncclGetUniqueId"));
    if (!get) fail(HFB_CUDA, "libnccl.so.2 lacks ncclGetUniqueId");
    NcclId id;
    nccl_check(get(&id), "ncclGetUniqueId");
    std::memcpy(out128, id.internal, sizeof id.internal);
  });
}

}  // extern "C"

// ---- peer-memory transport: export / attach ----------------------------------------
namespace {

constexpr char kPeerMagic[8] = {'H', 'F', 'B', 'P', 'E', 'E', 'R', '1'};
struct PeerBlobHead {
  char magic[8];
  int32_t rank, nranks, device, nfields;
  int64_t nx, ny;
  cudaIpcMemHandle_t sig;
  cudaIpcMemHandle_t gather;
};
struct PeerBlobField {
  char name[48];
  int32_t nbuf, pad;
  int64_t pitch, plane, origin_off;
  cudaIpcMemHandle_t h[3];
};

}  // namespace

extern "C" {

hfb_status hfb_peer_export(hfb_ctx* c, void* buf, size_t cap, size_t* len) {
  return guarded([&] {
    if (!c || !c->app) fail(HFB_CONFIG, "no program loaded");
    if (!c->decomposed || c->decomp.px * c->decomp.py <= 1)
      fail(HFB_CONFIG, "peer transport needs a multi-rank decomposition");
    if (c->group) fail(HFB_CONFIG, "in-process groups exchange halos by device copies");
    cudaSetDevice(c->device);
    if (!c->peer_sig) {
      cuda_check(cudaMalloc(&c->peer_sig, kSigWords * sizeof(uint64_t)), "cudaMalloc(signals)");
      cuda_check(cudaMemset(c->peer_sig, 0, kSigWords * sizeof(uint64_t)), "cudaMemset");
      // ordered reductions: every rank's column partials in global (j, i) order, two
      // parities (a 2-D plane per rank: small next to the 3-D fields)
      const size_t g = 2 * static_cast<size_t>(c->decomp.global_nx * c->decomp.global_ny);
      cuda_check(cudaMalloc(&c->peer_gather, g * sizeof(double)), "cudaMalloc(gather)");
      cuda_check(cudaMemset(c->peer_gather, 0, g * sizeof(double)), "cudaMemset");
    }
    // every bound array gets its device buffers now (double-buffered fields: all three
    // stage buffers), so the neighbours can map them before the first step
    std::vector<PeerBlobField> fs;
    for (auto& [name, s] : c->slots) {
      if (!s.host) continue;
      check_bounds(c, s);
      ensure_device(c, s, s.decl->pingpong, s.decl->pingpong ? 3 : 1);
      PeerBlobField f{};
      if (name.size() >= sizeof f.name) fail(HFB_CONFIG, "array name '%s' too long", name.c_str());
      std::strncpy(f.name, name.c_str(), sizeof f.name - 1);
      for (int b = 0; b < 3; ++b) {
        if (!s.dev[b]) break;
        cuda_check(cudaIpcGetMemHandle(&f.h[b], s.dev[b]), "cudaIpcGetMemHandle");
        f.nbuf = b + 1;
      }
      f.pitch = s.lay.pitch;
      f.plane = s.lay.plane;
      f.origin_off = s.lay.origin_off;
      fs.push_back(f);
    }
    // the ASUCA scheme's exchanged scratch (fu, fv: the slow momentum tendencies, pa: the
    // RK2 midpoint pressure), when the scheme's parameters are set: allocated now so the
    // neighbours map them before the first step
    auto ns = c->scalars.find("nsound");
    if (c->app->app == "dycore" && !c->app->plugin && ns != c->scalars.end() && ns->second.init) {
      asuca_prepare(c);
      const Slot& th = slot(c, "th");
      const std::pair<const char*, double*> scr[3] = {
          {"asu:fu", c->asu[2]}, {"asu:fv", c->asu[3]}, {"asu:pa", c->asu[5]}};
      for (const auto& [nm, base] : scr) {
        PeerBlobField f{};
        std::strncpy(f.name, nm, sizeof f.name - 1);
        cuda_check(cudaIpcGetMemHandle(&f.h[0], base), "cudaIpcGetMemHandle");
        f.nbuf = 1;
        f.pitch = th.lay.pitch;
        f.plane = th.lay.plane;
        f.origin_off = th.lay.origin_off;
        fs.push_back(f);
      }
      c->asu_exported = true;
    }
    cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    PeerBlobHead h{};
    std::memcpy(h.magic, kPeerMagic, 8);
    h.rank = c->decomp.rank;
    h.nranks = c->decomp.px * c->decomp.py;
    h.device = c->device;
    h.nfields = static_cast<int32_t>(fs.size());
    h.nx = c->decomp.nx;
    h.ny = c->decomp.ny;
    cuda_check(cudaIpcGetMemHandle(&h.sig, c->peer_sig), "cudaIpcGetMemHandle(signals)");
    cuda_check(cudaIpcGetMemHandle(&h.gather, c->peer_gather), "cudaIpcGetMemHandle(gather)");
    const size_t need = sizeof h + fs.size() * sizeof(PeerBlobField);
    *len = need;
    if (!buf) return;
    if (cap < need) fail(HFB_CONFIG, "peer blob needs %zu bytes", need);
    std::memcpy(buf, &h, sizeof h);
    if (!fs.empty())
      std::memcpy(static_cast<char*>(buf) + sizeof h, fs.data(), fs.size() * sizeof(PeerBlobField));
  });
}

hfb_status hfb_peer_stats(hfb_ctx* c, int64_t* pushes, int64_t* handoffs) {
  return guarded([&] {
    if (!c) fail(HFB_CONFIG, "null context");
    if (pushes) *pushes = c->peer_pushes;
    if (handoffs) *handoffs = c->peer_handoffs;
  });
}

hfb_status hfb_peer_attach(hfb_ctx* c, int n, const void* const* blobs, const size_t* lens) {
  return guarded([&] {
    if (!c || !c->peer_sig) fail(HFB_CONFIG, "hfb_peer_export first");
    if (c->peer) fail(HFB_CONFIG, "peers are already attached to this context");
    const hfb_decomp& d = c->decomp;
    if (n != d.px * d.py) fail(HFB_CONFIG, "%d blobs for %d ranks", n, d.px * d.py);
    cudaSetDevice(c->device);
    std::vector<PeerRank> peers(static_cast<size_t>(n));
    std::vector<bool> seen(static_cast<size_t>(n), false);
    auto open = [&](const cudaIpcMemHandle_t& hd) {
      void* p = nullptr;
      cuda_check(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess),
                 "cudaIpcOpenMemHandle");
      c->ipc_opened.push_back(p);
      return p;
    };
    for (int q = 0; q < n; ++q) {
      if (lens[q] < sizeof(PeerBlobHead)) fail(HFB_CONFIG, "peer blob %d truncated", q);
      PeerBlobHead h;
      std::memcpy(&h, blobs[q], sizeof h);
      if (std::memcmp(h.magic, kPeerMagic, 8) != 0) fail(HFB_CONFIG, "blob %d is not a peer blob", q);
      if (h.nranks != n || h.rank < 0 || h.rank >= n || seen[h.rank])
        fail(HFB_CONFIG, "blob %d: rank %d of %d (duplicate or out of range)", q, h.rank, h.nranks);
      seen[h.rank] = true;
      if (lens[q] != sizeof h + static_cast<size_t>(h.nfields) * sizeof(PeerBlobField))
        fail(HFB_CONFIG, "peer blob %d has a bad length", q);
      if (h.rank == d.rank) continue;
      PeerRank& pr = peers[h.rank];
      pr.nx = h.nx;
      pr.ny = h.ny;
      pr.sig = static_cast<uint64_t*>(open(h.sig));
      pr.gather = static_cast<double*>(open(h.gather));
      const int rx = h.rank % d.px, ry = h.rank / d.px;
      if (std::abs(rx - d.rx) > 1 || std::abs(ry - d.ry) > 1) continue;  // not a neighbour
      const char* fp = static_cast<const char*>(blobs[q]) + sizeof h;
      for (int f = 0; f < h.nfields; ++f) {
        PeerBlobField bf;
        std::memcpy(&bf, fp + f * sizeof bf, sizeof bf);
        PeerField pf;
        pf.nbuf = bf.nbuf;
        pf.pitch = bf.pitch;
        pf.plane = bf.plane;
        pf.origin_off = bf.origin_off;
        for (int b = 0; b < bf.nbuf && b < 3; ++b) pf.base[b] = static_cast<double*>(open(bf.h[b]));
        pr.fields[bf.name] = pf;
      }
    }
    c->peers = std::move(peers);
    c->peer = true;
  });
}

}  // extern "C"

// ===========================================================================
// State I/O and scenario files.
//
// The reference's harness input is "a scenario file naming the program, array shapes,
// fill patterns (constant, linear ramp, seeded pseudo-random with stated algorithm and
// seed), and expected-checksum entries" (never implemented: scenario.cpp:1
// is a placeholder). HFBSTAT1 images are the matching binary MachineState dump: program,
// scalars, array bounds and data in the reference's ArrayValue order (row-major, last
// subscript fastest, interp.cpp:485-494), so an image is independent of the device
// layout and of the caller's host order, and the oracle (tests/, oracle/) reads and
// writes the same bytes (paper_1710_08616_b200/state.py).
//
// HFBSTAT1 (little-endian): "HFBSTAT1" | u32 version=1 | str program | str module |
//   u32 nscalars | { str name | u8 type (0 int, 1 real) | u8 set | 8-byte value } |
//   u32 narrays | { str name | u32 rank | i64 lower[rank] | i64 upper[rank] |
//                   f64 data[count] } | u64 FNV-1a 64 of every preceding byte
// where str = u32 length + bytes.
// ===========================================================================
namespace {

constexpr char kStateMagic[8] = {'H', 'F', 'B', 'S', 'T', 'A', 'T', '1'};

uint64_t fnv1a(uint64_t h, const void* p, size_t n) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t q = 0; q < n; ++q) {
    h ^= b[q];
    h *= 0x100000001b3ull;
  }
  return h;
}
constexpr uint64_t kFnvBasis = 0xcbf29ce484222325ull;

void rowmajor_strides(const Slot& s, int64_t st[4]) {
  int64_t acc = 1;
  for (int d = s.rank - 1; d >= 0; --d) {
    const int64_t e = s.upper[d] - s.lower[d] + 1;
    st[d] = e > 1 ? acc : 0;
    acc *= e;
  }
}

// visit every element: f(flat index in ArrayValue order, element offset in the host buffer)
template <class F>
void for_each_element(const Slot& s, F&& f) {
  int64_t ext[4] = {1, 1, 1, 1}, idx[4] = {0, 0, 0, 0};
  for (int d = 0; d < s.rank; ++d) ext[d] = s.upper[d] - s.lower[d] + 1;
  for (int64_t flat = 0; flat < s.count; ++flat) {
    int64_t off = 0;
    for (int d = 0; d < s.rank; ++d) off += idx[d] * s.hstride[d];
    f(flat, off);
    for (int d = s.rank - 1; d >= 0; --d) {  // odometer, last subscript fastest
      if (++idx[d] < ext[d]) break;
      idx[d] = 0;
    }
  }
}

// the newest copy of a bound array in ArrayValue order; residency is left unchanged
std::vector<double> read_newest(hfb_ctx* c, Slot& s) {
  check_bounds(c, s);
  std::vector<double> out(static_cast<size_t>(s.count));
  if (s.has_device && s.res == kDevice) {
    Slot t = s;
    rowmajor_strides(s, t.hstride);
    const size_t bytes = static_cast<size_t>(s.count) * sizeof(double);
    ensure_staging(c, bytes);
    cuda_check(launch_relayout(s.d(), c->staging, relayout_of(t), false, c->stream),
               "relayout(D2H)");
    cuda_check(cudaMemcpyAsync(out.data(), c->staging, bytes, cudaMemcpyDeviceToHost, c->stream),
               "cudaMemcpyAsync(D2H)");
    cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  } else {
    for_each_element(s, [&](int64_t flat, int64_t off) { out[flat] = s.host[off]; });
  }
  return out;
}

// write ArrayValue-ordered data into the slot's host buffer, binding a context-owned one
// (pinned) when none is bound; the host copy becomes the newest
void write_host(hfb_ctx* c, Slot& s, int rank, const int64_t* lo, const int64_t* hi,
                const double* data) {
  if (!s.host) {
    int64_t count = 1;
    for (int d = 0; d < rank; ++d) count *= hi[d] - lo[d] + 1;
    double* buf = nullptr;
    cudaSetDevice(c->device);
    cuda_check(cudaMallocHost(&buf, static_cast<size_t>(count) * sizeof(double)),
               "cudaMallocHost(state array)");
    s.owned = buf;
    hfb_status rc = hfb_bind_array(c, s.module.c_str(), s.name.c_str(), rank, lo, hi, buf,
                                   nullptr, 0);
    if (rc != HFB_OK) fail(rc, "%s", hfb_last_error());
  } else {
    if (rank != s.rank) fail(HFB_RUNTIME, "array '%s': rank %d vs bound rank %d", s.name.c_str(),
                             rank, s.rank);
    for (int d = 0; d < rank; ++d)
      if (lo[d] != s.lower[d] || hi[d] != s.upper[d])
        fail(HFB_RUNTIME, "array '%s' is bound with bounds [%lld:%lld] in dimension %d, the "
                          "state has [%lld:%lld]", s.name.c_str(), (long long)s.lower[d],
             (long long)s.upper[d], d + 1, (long long)lo[d], (long long)hi[d]);
  }
  for_each_element(s, [&](int64_t flat, int64_t off) { s.host[off] = data[flat]; });
  if (s.has_device) s.res = kHost;  // host newer than the device copy
}

struct Writer {
  FILE* f;
  uint64_t h = kFnvBasis;
  void put(const void* p, size_t n) {
    if (fwrite(p, 1, n, f) != n) fail(HFB_IO, "write error");
    h = fnv1a(h, p, n);
  }
  template <class T>
  void pod(T v) { put(&v, sizeof v); }
  void str(const std::string& s) {
    pod<uint32_t>(static_cast<uint32_t>(s.size()));
    put(s.data(), s.size());
  }
};

struct Reader {
  FILE* f;
  std::string path;
  uint64_t h = kFnvBasis;
  void get(void* p, size_t n) {
    if (fread(p, 1, n, f) != n) fail(HFB_IO, "'%s': truncated state image", path.c_str());
    h = fnv1a(h, p, n);
  }
  template <class T>
  T pod() {
    T v;
    get(&v, sizeof v);
    return v;
  }
  std::string str() {
    const uint32_t n = pod<uint32_t>();
    if (n > 4096) fail(HFB_IO, "'%s': corrupt state image (name length %u)", path.c_str(), n);
    std::string s(n, '\0');
    get(&s[0], n);
    return s;
  }
};

struct FileCloser {
  FILE* f;
  ~FileCloser() {
    if (f) fclose(f);
  }
};

void save_state(hfb_ctx* c, const char* path) {
  if (!c || !c->app) fail(HFB_CONFIG, "no program loaded");
  cudaSetDevice(c->device);
  FILE* f = fopen(path, "wb");
  if (!f) fail(HFB_IO, "cannot open '%s' for writing", path);
  FileCloser fc{f};
  Writer w{f};
  w.put(kStateMagic, 8);
  w.pod<uint32_t>(1);
  w.str(c->app->app);
  w.str(c->app->module);
  w.pod<uint32_t>(static_cast<uint32_t>(c->scalars.size()));
  for (const auto& [name, v] : c->scalars) {
    w.str(name);
    w.pod<uint8_t>(v.type == SType::Int ? 0 : 1);
    w.pod<uint8_t>(v.init ? 1 : 0);
    if (v.type == SType::Int)
      w.pod<int64_t>(v.i);
    else
      w.pod<double>(v.r);
  }
  uint32_t nbound = 0;
  for (const auto& [name, s] : c->slots) nbound += s.host ? 1 : 0;
  w.pod<uint32_t>(nbound);
  for (auto& [name, s] : c->slots) {
    if (!s.host) continue;
    std::vector<double> data = read_newest(c, s);
    w.str(name);
    w.pod<uint32_t>(static_cast<uint32_t>(s.rank));
    for (int d = 0; d < s.rank; ++d) w.pod<int64_t>(s.lower[d]);
    for (int d = 0; d < s.rank; ++d) w.pod<int64_t>(s.upper[d]);
    w.put(data.data(), data.size() * sizeof(double));
  }
  const uint64_t sum = w.h;
  if (fwrite(&sum, 1, sizeof sum, f) != sizeof sum) fail(HFB_IO, "write error on '%s'", path);
  if (fflush(f) != 0) fail(HFB_IO, "write error on '%s'", path);
}

void load_state(hfb_ctx* c, const char* path) {
  if (!c) fail(HFB_CONFIG, "null context");
  FILE* f = fopen(path, "rb");
  if (!f) fail(HFB_IO, "cannot open '%s'", path);
  FileCloser fc{f};
  Reader r{f, path};
  char magic[8];
  r.get(magic, 8);
  if (std::memcmp(magic, kStateMagic, 8) != 0) fail(HFB_IO, "'%s' is not an HFBSTAT1 image", path);
  const uint32_t version = r.pod<uint32_t>();
  if (version != 1) fail(HFB_IO, "'%s': unsupported state image version %u", path, version);
  const std::string app = r.str(), module = r.str();
  if (!c->app) {
    hfb_status rc = hfb_load_program(c, app.c_str());
    if (rc != HFB_OK) fail(rc, "%s", hfb_last_error());
  } else if (c->app->app != app) {
    fail(HFB_CONFIG, "state image of program '%s' loaded into a context holding '%s'",
         app.c_str(), c->app->app.c_str());
  }
  if (module != c->app->module) fail(HFB_IO, "'%s': module '%s' is not '%s'", path,
                                     module.c_str(), c->app->module.c_str());
  // read everything first, apply after the checksum verified
  struct SV { std::string name; uint8_t type, set; int64_t i; double r; };
  std::vector<SV> scal(r.pod<uint32_t>());
  for (SV& v : scal) {
    v.name = r.str();
    v.type = r.pod<uint8_t>();
    v.set = r.pod<uint8_t>();
    if (v.type == 0) v.i = r.pod<int64_t>(); else v.r = r.pod<double>();
  }
  struct AV { std::string name; int rank; int64_t lo[4], hi[4]; std::vector<double> data; };
  std::vector<AV> arrs(r.pod<uint32_t>());
  for (AV& a : arrs) {
    a.name = r.str();
    a.rank = static_cast<int>(r.pod<uint32_t>());
    if (a.rank < 1 || a.rank > 4) fail(HFB_IO, "'%s': array '%s' has rank %d", path,
                                       a.name.c_str(), a.rank);
    int64_t count = 1;
    for (int d = 0; d < a.rank; ++d) a.lo[d] = r.pod<int64_t>();
    for (int d = 0; d < a.rank; ++d) {
      a.hi[d] = r.pod<int64_t>();
      if (a.hi[d] < a.lo[d]) fail(HFB_IO, "'%s': array '%s' has an empty dimension", path,
                                  a.name.c_str());
      count *= a.hi[d] - a.lo[d] + 1;
    }
    if (count > (int64_t(1) << 34)) fail(HFB_IO, "'%s': array '%s' too large", path, a.name.c_str());
    a.data.resize(static_cast<size_t>(count));
    r.get(a.data.data(), a.data.size() * sizeof(double));
  }
  const uint64_t expect = r.h;
  uint64_t stored = 0;
  if (fread(&stored, 1, sizeof stored, f) != sizeof stored || stored != expect)
    fail(HFB_IO, "'%s': checksum mismatch (corrupt or truncated state image)", path);
  for (const SV& v : scal) {
    auto it = c->scalars.find(v.name);
    if (it == c->scalars.end()) fail(HFB_IO, "'%s': unknown scalar '%s'", path, v.name.c_str());
    Scalar& s = it->second;
    if ((s.type == SType::Int) != (v.type == 0))
      fail(HFB_IO, "'%s': scalar '%s' has the wrong type", path, v.name.c_str());
    s.init = v.set != 0;
    if (v.type == 0) { s.i = v.i; s.r = static_cast<double>(v.i); }
    else { s.r = v.r; s.i = static_cast<int64_t>(v.r); }
  }
  for (const AV& a : arrs) {
    Slot& s = slot_ref(c, c->app->module, a.name);
    if (a.rank != static_cast<int>(s.decl->dims.size()))
      fail(HFB_IO, "'%s': array '%s' has rank %d, declared %zu", path, a.name.c_str(), a.rank,
           s.decl->dims.size());
    write_host(c, s, a.rank, a.lo, a.hi, a.data.data());
  }
}

// ---- scenario files -------------------------------------------------------------------
//   program <app>            entry <routine>          set <scalar> <value>
//   option reduction ordered|fast (hfb_set_reduction_order)
//   array <name> <dims...>   (dims: lo:hi or n; default: the declaration, evaluated)
//   fill <name> const <v> | ramp <a> <b> | splitmix <seed> <offset> <scale>
//   expect <array> sum <value> <rel_tol> | expect <array> bits <hex>
//   expect <scalar> value <value> <rel_tol>
// '#' starts a comment. splitmix: offset + scale * u, u = (splitmix64((seed << 40) + flat)
// >> 11) * 2^-53 with the reference's SplitMix64 (interp.cpp:22-28) over the ArrayValue
// flat index; ramp: a + b * flat.
uint64_t splitmix64(uint64_t x) {  // interp.cpp:22-28
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

std::vector<std::string> split_ws(const std::string& line) {
  std::vector<std::string> t;
  size_t q = 0;
  while (q < line.size()) {
    while (q < line.size() && std::isspace(static_cast<unsigned char>(line[q]))) ++q;
    if (q >= line.size() || line[q] == '#') break;
    size_t e = q;
    while (e < line.size() && !std::isspace(static_cast<unsigned char>(line[e]))) ++e;
    t.push_back(line.substr(q, e - q));
    q = e;
  }
  return t;
}

double num(const std::string& s, const char* what, int ln) {
  char* end = nullptr;
  double v = std::strtod(s.c_str(), &end);
  if (s.empty() || *end != '\0') fail(HFB_IO, "scenario line %d: bad %s '%s'", ln, what, s.c_str());
  return v;
}

void run_scenario(hfb_ctx* c, const char* path, hfb_launch_stats* stats, std::string& report) {
  if (!c) fail(HFB_CONFIG, "null context");
  FILE* f = fopen(path, "r");
  if (!f) fail(HFB_IO, "cannot open scenario '%s'", path);
  std::vector<std::pair<int, std::vector<std::string>>> lines;
  {
    FileCloser fc{f};
    char buf[4096];
    int ln = 0;
    while (fgets(buf, sizeof buf, f)) {
      ++ln;
      auto t = split_ws(buf);
      if (!t.empty()) lines.push_back({ln, t});
    }
  }
  std::string entry = "main";
  struct Fill { std::string kind; double a = 0, b = 0; uint64_t seed = 0; };
  std::map<std::string, std::vector<std::pair<int64_t, int64_t>>> shapes;
  std::vector<std::pair<std::string, Fill>> fills;
  struct Expect { int ln; std::string name, kind, a, b; };
  std::vector<Expect> expects;
  for (auto& lt : lines) {
    const int ln = lt.first;
    const std::vector<std::string>& t = lt.second;
    const std::string& k = t[0];
    auto need = [&](size_t n) {
      if (t.size() != n) fail(HFB_IO, "scenario line %d: '%s' takes %zu fields", ln, k.c_str(),
                              n - 1);
    };
    if (k == "program") {
      need(2);
      if (!c->app) {
        hfb_status rc = hfb_load_program(c, t[1].c_str());
        if (rc != HFB_OK) fail(rc, "%s", hfb_last_error());
      } else if (c->app->app != lower(t[1].c_str())) {
        fail(HFB_CONFIG, "scenario program '%s' in a context holding '%s'", t[1].c_str(),
             c->app->app.c_str());
      }
    } else if (!c->app) {
      fail(HFB_IO, "scenario line %d: 'program' must come first", ln);
    } else if (k == "entry") {
      need(2);
      entry = t[1];
    } else if (k == "option") {  // option reduction ordered|fast
      need(3);
      if (t[1] != "reduction" || (t[2] != "ordered" && t[2] != "fast"))
        fail(HFB_IO, "scenario line %d: unknown option '%s %s'", ln, t[1].c_str(), t[2].c_str());
      c->reduce_ordered = t[2] == "ordered";
    } else if (k == "set") {
      need(3);
      Scalar& s = scalar_ref(c, c->app->module, lower(t[1].c_str()));
      const double v = num(t[2], "value", ln);
      s.r = v;
      s.i = static_cast<int64_t>(v);
      if (s.type == SType::Int && static_cast<double>(s.i) != v)
        fail(HFB_IO, "scenario line %d: integer scalar '%s' set to %s", ln, t[1].c_str(),
             t[2].c_str());
      s.init = true;
    } else if (k == "array") {
      if (t.size() < 3 || t.size() > 6) fail(HFB_IO, "scenario line %d: array <name> <dims>", ln);
      std::vector<std::pair<int64_t, int64_t>> dims;
      for (size_t q = 2; q < t.size(); ++q) {
        const size_t colon = t[q].find(':');
        if (colon == std::string::npos)
          dims.push_back({1, static_cast<int64_t>(num(t[q], "extent", ln))});
        else
          dims.push_back({static_cast<int64_t>(num(t[q].substr(0, colon), "bound", ln)),
                          static_cast<int64_t>(num(t[q].substr(colon + 1), "bound", ln))});
      }
      shapes[lower(t[1].c_str())] = dims;
    } else if (k == "fill") {
      if (t.size() < 3) fail(HFB_IO, "scenario line %d: fill <name> <kind> ...", ln);
      Fill fl;
      fl.kind = t[2];
      if (fl.kind == "const") {
        need(4);
        fl.a = num(t[3], "value", ln);
      } else if (fl.kind == "ramp") {
        need(5);
        fl.a = num(t[3], "value", ln);
        fl.b = num(t[4], "value", ln);
      } else if (fl.kind == "splitmix") {
        need(6);
        fl.seed = std::strtoull(t[3].c_str(), nullptr, 0);
        fl.a = num(t[4], "offset", ln);
        fl.b = num(t[5], "scale", ln);
      } else {
        fail(HFB_IO, "scenario line %d: unknown fill '%s'", ln, fl.kind.c_str());
      }
      fills.push_back({lower(t[1].c_str()), fl});
    } else if (k == "expect") {
      if (t.size() < 4 || t.size() > 5) fail(HFB_IO, "scenario line %d: expect <name> <kind> ...", ln);
      expects.push_back({ln, lower(t[1].c_str()), t[2], t[3], t.size() > 4 ? t[4] : "0"});
    } else {
      fail(HFB_IO, "scenario line %d: unknown keyword '%s'", ln, k.c_str());
    }
  }
  if (!c->app) fail(HFB_IO, "scenario '%s' names no program", path);
  // bind every filled array to a context-owned buffer and fill it (ArrayValue order)
  for (auto& [name, fl] : fills) {
    Slot& s = slot_ref(c, c->app->module, name);
    std::vector<std::pair<int64_t, int64_t>> dims;
    auto it = shapes.find(name);
    if (it != shapes.end()) {
      dims = it->second;
    } else {
      for (auto& d : s.decl->dims) dims.push_back({eval_dim(c, d.first), eval_dim(c, d.second)});
    }
    const int rank = static_cast<int>(dims.size());
    int64_t lo[4], hi[4], count = 1;
    for (int d = 0; d < rank; ++d) {
      lo[d] = dims[d].first;
      hi[d] = dims[d].second;
      count *= hi[d] - lo[d] + 1;
    }
    std::vector<double> data(static_cast<size_t>(count));
    for (int64_t q = 0; q < count; ++q) {
      if (fl.kind == "const") {
        data[q] = fl.a;
      } else if (fl.kind == "ramp") {
        data[q] = fl.a + fl.b * static_cast<double>(q);
      } else {
        const double u =
            static_cast<double>(splitmix64((fl.seed << 40) + static_cast<uint64_t>(q)) >> 11) *
            0x1.0p-53;
        data[q] = fl.a + fl.b * u;
      }
    }
    // a caller buffer stays bound (same bounds required); a context-owned buffer of
    // another size is replaced
    if (s.owned && s.count != count) {
      if (s.has_device) fail(HFB_CONFIG, "scenario reshapes '%s' after a transfer", name.c_str());
      cudaFreeHost(s.owned);
      s.owned = nullptr;
      s.host = nullptr;
    }
    write_host(c, s, rank, lo, hi, data.data());
  }
  hfb_status rc = hfb_run(c, entry.c_str(), stats);
  if (rc != HFB_OK) fail(rc, "%s", hfb_last_error());
  // expectations
  std::string first_fail;
  char line[512];
  for (const Expect& e : expects) {
    bool ok = false;
    if (e.kind == "sum" || e.kind == "bits") {
      Slot& s = slot_ref(c, c->app->module, e.name);
      std::vector<double> data = read_newest(c, s);
      if (e.kind == "sum") {
        double sum = 0.0;
        for (double v : data) sum += v;
        const double want = num(e.a, "value", e.ln), tol = num(e.b, "tolerance", e.ln);
        ok = tol == 0.0 ? sum == want : std::fabs(sum - want) <= tol * std::fabs(want);
        snprintf(line, sizeof line, "%s sum %.17g expected %.17g (rel tol %g) %s\n",
                 e.name.c_str(), sum, want, tol, ok ? "ok" : "FAIL");
      } else {
        const uint64_t h = fnv1a(kFnvBasis, data.data(), data.size() * sizeof(double));
        const uint64_t want = std::strtoull(e.a.c_str(), nullptr, 0);
        ok = h == want;
        snprintf(line, sizeof line, "%s bits 0x%016llx expected 0x%016llx %s\n", e.name.c_str(),
                 (unsigned long long)h, (unsigned long long)want, ok ? "ok" : "FAIL");
      }
    } else if (e.kind == "value") {
      const double v = rval(c, e.name.c_str());
      const double want = num(e.a, "value", e.ln), tol = num(e.b, "tolerance", e.ln);
      ok = tol == 0.0 ? v == want : std::fabs(v - want) <= tol * std::fabs(want);
      snprintf(line, sizeof line, "%s value %.17g expected %.17g (rel tol %g) %s\n",
               e.name.c_str(), v, want, tol, ok ? "ok" : "FAIL");
    } else {
      fail(HFB_IO, "scenario line %d: unknown expectation '%s'", e.ln, e.kind.c_str());
    }
    report += line;
    if (!ok && first_fail.empty()) first_fail = line;
  }
  if (!first_fail.empty()) {
    if (!first_fail.empty() && first_fail.back() == '\n') first_fail.pop_back();
    fail(HFB_VALIDATION, "scenario '%s': %s", path, first_fail.c_str());
  }
}

}  // namespace

extern "C" {

hfb_status hfb_save_state(hfb_ctx* c, const char* path) {
  return guarded([&] { save_state(c, path); });
}

hfb_status hfb_load_state(hfb_ctx* c, const char* path) {
  return guarded([&] { load_state(c, path); });
}

hfb_status hfb_host_array(hfb_ctx* c, const char* module, const char* name, double** host,
                          int* rank, int64_t lower_out[4], int64_t upper_out[4],
                          int64_t strides[4]) {
  return guarded([&] {
    Slot& s = slot_ref(c, lower(module), lower(name));
    if (!s.host) fail(HFB_CONFIG, "array '%s' of module '%s' is not bound", name, module);
    *host = s.host;
    *rank = s.rank;
    for (int d = 0; d < 4; ++d) {
      lower_out[d] = d < s.rank ? s.lower[d] : 1;
      upper_out[d] = d < s.rank ? s.upper[d] : 1;
      strides[d] = d < s.rank ? s.hstride[d] : 0;
    }
  });
}

hfb_status hfb_array_checksum(hfb_ctx* c, const char* module, const char* name, double* sum,
                              uint64_t* bits) {
  return guarded([&] {
    Slot& s = slot_ref(c, lower(module), lower(name));
    cudaSetDevice(c->device);
    std::vector<double> data = read_newest(c, s);
    double acc = 0.0;
    for (double v : data) acc += v;
    if (sum) *sum = acc;
    if (bits) *bits = fnv1a(kFnvBasis, data.data(), data.size() * sizeof(double));
  });
}

hfb_status hfb_run_scenario(hfb_ctx* c, const char* path, hfb_launch_stats* stats, char* report,
                            size_t report_len) {
  std::string rep;
  hfb_status rc = guarded([&] {
    if (c) cudaSetDevice(c->device);
    run_scenario(c, path, stats, rep);
  });
  if (report && report_len) {
    std::strncpy(report, rep.c_str(), report_len - 1);
    report[report_len - 1] = '\0';
  }
  return rc;
}

}  // extern "C"

extern "C" {

hfb_status hfb_plugin_prepare(hfb_ctx* c, const char* name, int mode) {
  return guarded([&] {
    if (is_scratch(name)) return;
    if (mode == 0)
      dev_read(c, name);
    else
      dev_write(c, name);
  });
}

hfb_status hfb_plugin_written(hfb_ctx* c, const char* name) {
  return guarded([&] {
    if (is_scratch(name)) return;
    dev_written(c, name);
    // a checked program sets the flags of exactly the elements it writes; an unchecked
    // one is only known to have written the array: count it as set
    if (!c->plugin_tracks_init) init_written(c, name);
  });
}

hfb_status hfb_plugin_view(hfb_ctx* c, const char* name, hfb_view* out) {
  return guarded([&] {
    if (is_scratch(name)) {
      auto it = c->scratch.find(name);
      if (it == c->scratch.end()) fail(HFB_CONFIG, "no scratch array '%s'", name);
      const Scratch& sa = it->second;
      fill_view(sa.lay, sa.roles, sa.rank, sa.lower, sa.dev + sa.lay.origin_off, out);
      return;
    }
    Slot& s = slot(c, name);
    if (!s.has_device) fail(HFB_RESIDENCY, "array '%s' has no device copy (missing transfer)", name);
    Role roles[4];
    for (int q = 0; q < s.rank; ++q) roles[q] = s.decl->roles[q];
    fill_view(s.lay, roles, s.rank, s.lower, s.d(), out);
  });
}

hfb_status hfb_plugin_host(hfb_ctx* c, const char* name, int write, hfb_view* out) {
  return guarded([&] {
    if (is_scratch(name))
      fail(HFB_CONFIG, "host access to the routine-local array '%s' is not supported", name);
    Slot& s = slot(c, name);
    check_bounds(c, s);
    // host-code access checks (slot_side, interp.cpp:406-409)
    if (!write && s.res == kDevice)
      fail(HFB_RESIDENCY, "host copy of '%s' is stale (device copy was modified)", name);
    if (write && s.has_device) s.res = kHost;
    out->origin = s.host;
    for (int d = 0; d < 4; ++d) {
      out->stride[d] = d < s.rank ? s.hstride[d] : 0;
      out->lower[d] = d < s.rank ? s.lower[d] : 1;
    }
  });
}

hfb_status hfb_plugin_host_ref(hfb_ctx* c, const char* name, hfb_host_ref* out) {
  return guarded([&] {
    if (is_scratch(name))
      fail(HFB_CONFIG, "host access to the routine-local array '%s' is not supported", name);
    Slot& s = slot(c, name);
    check_bounds(c, s);
    out->view.origin = s.host;
    for (int d = 0; d < 4; ++d) {
      out->view.stride[d] = d < s.rank ? s.hstride[d] : 0;
      out->view.lower[d] = d < s.rank ? s.lower[d] : 1;
    }
    static_assert(sizeof(s.res) == sizeof(int32_t), "residency word");
    out->residency = reinterpret_cast<int32_t*>(&s.res);
    out->has_device = &s.has_device;
  });
}

hfb_status hfb_plugin_array_info(hfb_ctx* c, const char* name, int* rank, int64_t lower[4],
                                 int64_t upper[4], uint8_t** dinit, uint8_t** hinit) {
  return guarded([&] {
    if (is_scratch(name)) {
      auto it = c->scratch.find(name);
      if (it == c->scratch.end()) fail(HFB_CONFIG, "no scratch array '%s'", name);
      Scratch& sa = it->second;
      if (!sa.dinit) {
        cuda_check(cudaMalloc(&sa.dinit, static_cast<size_t>(sa.lay.alloc_elems)),
                   "cudaMalloc(init)");
        cuda_check(cudaMemsetAsync(sa.dinit, 0, static_cast<size_t>(sa.lay.alloc_elems),
                                   c->stream),
                   "cudaMemsetAsync(init)");
      }
      *rank = sa.rank;
      for (int q = 0; q < 4; ++q) {
        lower[q] = q < sa.rank ? sa.lower[q] : 1;
        upper[q] = q < sa.rank ? sa.upper[q] : 1;
      }
      *dinit = sa.dinit + sa.lay.origin_off;
      *hinit = nullptr;
      return;
    }
    Slot& s = slot(c, name);
    check_bounds(c, s);
    c->plugin_tracks_init = true;
    *rank = s.rank;
    for (int q = 0; q < 4; ++q) {
      lower[q] = q < s.rank ? s.lower[q] : 1;
      upper[q] = q < s.rank ? s.upper[q] : 1;
    }
    *dinit = nullptr;
    if (s.has_device) {
      if (!s.dinit) ensure_dinit(c, s, 1);  // never tracked: defined
      *dinit = s.dinit + s.lay.origin_off;
    }
    *hinit = s.hinit;
  });
}

hfb_status hfb_plugin_scratch_clear_init(hfb_ctx* c, const char* key) {
  return guarded([&] {
    auto it = c->scratch.find(key);
    if (it == c->scratch.end()) fail(HFB_CONFIG, "no scratch array '%s'", key);
    Scratch& sa = it->second;
    if (sa.dinit)
      cuda_check(cudaMemsetAsync(sa.dinit, 0, static_cast<size_t>(sa.lay.alloc_elems), c->stream),
                 "cudaMemsetAsync(init)");
  });
}

hfb_status hfb_plugin_error(hfb_ctx* c, hfb_status status, const char* msg) {
  (void)c;
  return guarded([&] { fail(status, "%s", msg ? msg : "error"); });
}

hfb_status hfb_plugin_scratch(hfb_ctx* c, const char* key, int rank, const int64_t* lower,
                              const int64_t* upper, const int* roles) {
  return guarded([&] {
    if (rank < 1 || rank > 4) fail(HFB_CONFIG, "scratch '%s': rank %d", key, rank);
    Scratch& sa = c->scratch[key];
    bool same = sa.dev && sa.rank == rank;
    int64_t ext[4] = {1, 1, 1, 1};
    for (int q = 0; q < rank; ++q) {
      if (upper[q] < lower[q]) fail(HFB_RUNTIME, "scratch '%s': empty dimension %d", key, q + 1);
      same = same && sa.lower[q] == lower[q] && sa.upper[q] == upper[q] &&
             sa.roles[q] == static_cast<Role>(roles[q]);
      ext[roles[q]] *= upper[q] - lower[q] + 1;
    }
    if (same) return;
    if (sa.dev) cudaFree(sa.dev);
    if (sa.dinit) cudaFree(sa.dinit);
    sa.dev = nullptr;
    sa.dinit = nullptr;
    sa.rank = rank;
    for (int q = 0; q < rank; ++q) {
      sa.lower[q] = lower[q];
      sa.upper[q] = upper[q];
      sa.roles[q] = static_cast<Role>(roles[q]);
    }
    sa.lay = Layout::make(ext[kRoleI], ext[kRoleJ], ext[kRoleK], ext[kRoleL]);
    const size_t bytes = static_cast<size_t>(sa.lay.alloc_elems) * sizeof(double);
    cudaSetDevice(c->device);
    cuda_check(cudaMalloc(&sa.dev, bytes), "cudaMalloc(scratch)");
    cuda_check(cudaMemsetAsync(sa.dev, 0, bytes, c->stream), "cudaMemsetAsync");
  });
}

}  // extern "C"
