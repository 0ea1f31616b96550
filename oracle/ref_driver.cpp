// ref_driver.cpp — TEST INFRASTRUCTURE ONLY (oracle side). Never linked into the product.
//
// A thin command-line harness around the reference's own binary64 interpreter
// (`hft::interp`, /root/reference/proj/src/interp.cpp), compiled from the
// reference sources by oracle/Makefile into oracle/_ref/hft_ref. It plays the
// role of the scenario runner the reference specifies but never implemented
// (proj/src/scenario.cpp:1 is a placeholder):
//
//   * parses the .h90 sources (parser.hpp:10-15),
//   * for `mode gpu` runs the full pipeline build_model -> generate_target_tree
//     (CUDA-style) -> macro::expand -> re-parse (codegen.hpp:25-26, macro.hpp:45-46),
//   * allocates module arrays itself from the (expanded) declarations, working
//     around Program::elaborate_arrays (interp.cpp:1522-1561),
//   * fills inputs with the reference SplitMix64 (interp.cpp:22-28) indexed by the
//     logical row-major flat index (interp.cpp:485-494),
//   * runs run_reference / run_cpu_generated / run_gpu_simulated (interp.hpp:113-122),
//   * dumps arrays + scalars + LaunchStats to a small binary file read by
//     tests/hfb_dump.py.
//
// Scenario file format (one directive per line, '#' comments):
//   source <path.h90>                 (repeatable; order kept)
//   mode ref|cpu|gpu
//   entry <routine>                   (gpu mode: the hfd_ name, e.g. hfd_main)
//   backend cuda|acc                  (gpu mode code generator, codegen.hpp:9)
//   order forward|reverse|shuffled    (simulated thread order, interp.hpp:14)
//   shuffle_seed <u64>
//   max_steps <n>
//   family <acc_macro> <dom_macro>    (register an ordering-macro family, macro.hpp:28)
//   rotate <macro>                    (RotateLastToFront permutation for that family)
//   block <template|-> <x> <y> <z>    (block size per template suffix; '-' = default)
//   int  <module> <name> <value>
//   real <module> <name> <value>      (parsed with strtod; hex-float allowed)
//   fill <module> <name> <seed> <offset> <scale>   value = offset + scale*u(seed, flat)
//   unset <module> <name>             (allocated, init flags cleared)
//   dump <module> <name>              (array or scalar)
//   out <path>
//   repeat <n>                        (run the entry n times; for timing only)
//   app <program|plugin.so>           (mode b200: the engine program to run)
//   array <module> <name> <lo> <hi> [<lo> <hi> ...]   (mode b200 without sources: the
//                                     MachineState is built from the directives alone)
//
// Built with -DHFB_ADAPTER (oracle/_ref/hft_ref_b200), `mode b200` runs the entry on a
// B200 through integration/hfb_adapter.hpp — the reference-side drop-in for
// run_gpu_simulated — on the same MachineState the interpreter modes use.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "hft/analysis.hpp"
#include "hft/codegen.hpp"
#include "hft/diagnostics.hpp"
#include "hft/interp.hpp"
#include "hft/macro.hpp"
#include "hft/parser.hpp"
#include "hft/tokenize.hpp"
#ifdef HFB_ADAPTER
#include "hfb_adapter.hpp"
#endif

using namespace hft;

namespace {

struct FillSpec {
  std::string module, name;
  bool unset = false;
  uint64_t seed = 0;
  double offset = 0.0, scale = 1.0;
};

struct ScalarSet {
  std::string module, name;
  bool is_int = false;
  long long i = 0;
  double r = 0.0;
};

struct Scenario {
  std::vector<std::string> sources;
  std::string mode = "ref";
  bool acc_backend = false;
  std::string entry = "main";
  interp::ThreadOrder order = interp::ThreadOrder::Forward;
  uint64_t shuffle_seed = 0x5eed;
  long max_steps = 200L * 1000 * 1000;
  std::vector<std::pair<std::string, std::string>> families;
  std::vector<std::string> rotated;
  std::vector<std::pair<std::string, std::array<int, 3>>> blocks;
  std::vector<ScalarSet> scalars;
  std::vector<FillSpec> fills;
  std::vector<std::pair<std::string, std::string>> dumps;
  std::string out;
  int repeat = 1;
  std::string app;
  struct ArraySpec {
    std::string module, name;
    std::vector<long long> lo, hi;
  };
  std::vector<ArraySpec> arrays;
};

std::string read_text(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(ErrKind::Io, "cannot open '" + path + "'");
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

Scenario parse_scenario(const std::string& path) {
  Scenario sc;
  std::istringstream in(read_text(path));
  std::string line;
  while (std::getline(in, line)) {
    auto hash = line.find('#');
    if (hash != std::string::npos) line = line.substr(0, hash);
    std::istringstream ls(line);
    std::string cmd;
    if (!(ls >> cmd)) continue;
    if (cmd == "source") {
      std::string p;
      ls >> p;
      sc.sources.push_back(p);
    } else if (cmd == "mode") {
      ls >> sc.mode;
    } else if (cmd == "backend") {
      std::string b;
      ls >> b;
      sc.acc_backend = b == "acc";
    } else if (cmd == "entry") {
      ls >> sc.entry;
    } else if (cmd == "order") {
      std::string o;
      ls >> o;
      sc.order = o == "reverse"    ? interp::ThreadOrder::Reverse
                 : o == "shuffled" ? interp::ThreadOrder::Shuffled
                                   : interp::ThreadOrder::Forward;
    } else if (cmd == "shuffle_seed") {
      ls >> sc.shuffle_seed;
    } else if (cmd == "max_steps") {
      ls >> sc.max_steps;
    } else if (cmd == "family") {
      std::string a, d;
      ls >> a >> d;
      sc.families.emplace_back(a, d);
    } else if (cmd == "rotate") {
      std::string m;
      ls >> m;
      sc.rotated.push_back(m);
    } else if (cmd == "block") {
      std::string t;
      std::array<int, 3> b{};
      ls >> t >> b[0] >> b[1] >> b[2];
      sc.blocks.emplace_back(t == "-" ? "" : t, b);
    } else if (cmd == "int" || cmd == "real") {
      ScalarSet s;
      std::string v;
      ls >> s.module >> s.name >> v;
      s.is_int = cmd == "int";
      if (s.is_int)
        s.i = std::stoll(v);
      else
        s.r = std::strtod(v.c_str(), nullptr);
      sc.scalars.push_back(s);
    } else if (cmd == "fill") {
      FillSpec f;
      std::string off, scl;
      ls >> f.module >> f.name >> f.seed >> off >> scl;
      f.offset = std::strtod(off.c_str(), nullptr);
      f.scale = std::strtod(scl.c_str(), nullptr);
      sc.fills.push_back(f);
    } else if (cmd == "unset") {
      FillSpec f;
      f.unset = true;
      ls >> f.module >> f.name;
      sc.fills.push_back(f);
    } else if (cmd == "dump") {
      std::string m, n;
      ls >> m >> n;
      sc.dumps.emplace_back(m, n);
    } else if (cmd == "out") {
      ls >> sc.out;
    } else if (cmd == "repeat") {
      ls >> sc.repeat;
    } else if (cmd == "app") {
      ls >> sc.app;
    } else if (cmd == "array") {
      Scenario::ArraySpec a;
      ls >> a.module >> a.name;
      long long lo, hi;
      while (ls >> lo >> hi) {
        a.lo.push_back(lo);
        a.hi.push_back(hi);
      }
      sc.arrays.push_back(a);
    } else {
      fail(ErrKind::Config, "unknown scenario directive '" + cmd + "'");
    }
  }
  return sc;
}

// Minimal integer evaluator for declaration extents (module scalars, literals,
// + - * /). Mirrors what elaborate_arrays would do if it could see module
// scalars (interp.cpp:1531-1546).
long long eval_extent(const ast::Expr& e, interp::MachineState& st, const std::string& module) {
  using K = ast::Expr::Kind;
  switch (e.kind) {
    case K::IntLit: return e.int_value;
    case K::RealLit: return static_cast<long long>(e.real_value);
    case K::Var: {
      interp::ScalarValue* s = st.find_scalar(module, e.text);
      if (!s) s = st.find_scalar_any(e.text);
      if (!s || !s->initialized) fail(ErrKind::Config, "extent scalar '" + e.text + "' is unset");
      return s->type == ast::BaseType::Integer ? s->i : static_cast<long long>(s->r);
    }
    case K::Un: return -eval_extent(*e.args[0], st, module);
    case K::Bin: {
      long long a = eval_extent(*e.args[0], st, module);
      long long b = eval_extent(*e.args[1], st, module);
      switch (e.bin) {
        case ast::BinOp::Add: return a + b;
        case ast::BinOp::Sub: return a - b;
        case ast::BinOp::Mul: return a * b;
        case ast::BinOp::Div: return a / b;
        default: break;
      }
      break;
    }
    default: break;
  }
  fail(ErrKind::Config, "unsupported extent expression '" + ast::print_expr(e) + "'");
}

double unit_uniform(uint64_t seed, uint64_t flat) {
  // u(seed, flat) = (splitmix64((seed << 40) + flat) >> 11) * 2^-53
  return static_cast<double>(interp::splitmix64((seed << 40) + flat) >> 11) * 0x1.0p-53;
}

void allocate_arrays(const interp::Program& prog, interp::MachineState& st) {
  for (const auto& unit : prog.units())
    for (const ast::ModuleDecl& m : unit->modules) {
      auto& arrays = st.arrays[to_lower(m.name)];
      for (const ast::VarDecl& d : m.vars) {
        if (d.is_scalar()) continue;
        auto arr = std::make_shared<interp::ArrayValue>();
        arr->type = d.type;
        for (const ast::Dim& dim : d.dims) {
          long long lo = dim.lower ? eval_extent(*dim.lower, st, m.name) : 1;
          long long hi = eval_extent(*dim.upper, st, m.name);
          if (hi < lo) fail(ErrKind::Config, "non-positive extent for '" + d.name + "'");
          arr->lower.push_back(lo);
          arr->upper.push_back(hi);
        }
        size_t n = arr->size();
        arr->reals.assign(n, 0.0);
        arr->init.assign(n, 0);
        interp::ObjectSlot slot;
        slot.host = std::move(arr);
        arrays[to_lower(d.name)] = std::move(slot);
      }
    }
}

void put_u32(std::ofstream& o, uint32_t v) { o.write(reinterpret_cast<const char*>(&v), 4); }
void put_i64(std::ofstream& o, int64_t v) { o.write(reinterpret_cast<const char*>(&v), 8); }
void put_f64(std::ofstream& o, double v) { o.write(reinterpret_cast<const char*>(&v), 8); }
void put_str(std::ofstream& o, const std::string& s) {
  put_u32(o, static_cast<uint32_t>(s.size()));
  o.write(s.data(), static_cast<std::streamsize>(s.size()));
}

// mode b200 without sources: the MachineState from the scenario's own declarations
interp::MachineState state_from_directives(const Scenario& sc) {
  interp::MachineState st;
  for (const ScalarSet& s : sc.scalars) st.scalars[to_lower(s.module)][to_lower(s.name)] = {};
  for (const Scenario::ArraySpec& d : sc.arrays) {
    auto arr = std::make_shared<interp::ArrayValue>();
    arr->type = ast::BaseType::Real;
    arr->lower = d.lo;
    arr->upper = d.hi;
    arr->reals.assign(arr->size(), 0.0);
    arr->init.assign(arr->size(), 0);
    interp::ObjectSlot slot;
    slot.host = std::move(arr);
    st.arrays[to_lower(d.module)][to_lower(d.name)] = std::move(slot);
  }
  return st;
}

int run(const Scenario& sc) {
  std::vector<std::unique_ptr<ast::Unit>> units;
  for (const std::string& p : sc.sources)
    units.push_back(std::make_unique<ast::Unit>(parse_source(p, read_text(p))));

  std::unique_ptr<interp::Program> prog;
  if (sc.mode == "gpu") {
    codegen::TargetConfig cfg;
    cfg.architecture = Target::GPU;
    cfg.gpu_backend =
        sc.acc_backend ? codegen::GpuBackend::OpenAccStyle : codegen::GpuBackend::CudaStyle;
    for (const auto& [a, d] : sc.families) cfg.macros.register_family(a, d);
    for (const std::string& m : sc.rotated)
      cfg.macros.set_order(m, macro::PermSpec{macro::PermKind::RotateLastToFront, {}});
    for (const auto& [t, b] : sc.blocks) cfg.macros.set_block_size(t, b);
    analysis::ApplicationModel model = analysis::build_model(std::move(units));
    std::vector<codegen::GeneratedFile> files = codegen::generate_target_tree(model, cfg);
    std::vector<std::unique_ptr<ast::Unit>> gen;
    for (const codegen::GeneratedFile& f : files) {
      std::string expanded = macro::expand(f.text, cfg.macros, f.name);
      gen.push_back(std::make_unique<ast::Unit>(parse_source(f.name, expanded)));
    }
    prog = std::make_unique<interp::Program>(std::move(gen));
  } else if (sc.mode == "cpu") {
    codegen::TargetConfig cfg;
    cfg.architecture = Target::CPU;
    for (const auto& [a, d] : sc.families) cfg.macros.register_family(a, d);
    analysis::ApplicationModel model = analysis::build_model(std::move(units));
    std::vector<codegen::GeneratedFile> files = codegen::generate_target_tree(model, cfg);
    std::vector<std::unique_ptr<ast::Unit>> gen;
    for (const codegen::GeneratedFile& f : files) {
      std::string expanded = macro::expand(f.text, cfg.macros, f.name);
      gen.push_back(std::make_unique<ast::Unit>(parse_source(f.name, expanded)));
    }
    prog = std::make_unique<interp::Program>(std::move(gen));
  } else {
    prog = std::make_unique<interp::Program>(std::move(units));
  }

  const bool own_state = sc.mode == "b200" && sc.sources.empty();
  interp::MachineState st = own_state ? state_from_directives(sc) : prog->prepare_state();
  for (const ScalarSet& s : sc.scalars) {
    interp::ScalarValue* v = st.find_scalar(s.module, s.name);
    if (!v) fail(ErrKind::Config, "unknown scalar " + s.module + "." + s.name);
    if (s.is_int) {
      v->type = ast::BaseType::Integer;
      v->i = s.i;
    } else {
      v->type = ast::BaseType::Real;
      v->r = s.r;
    }
    v->initialized = true;
  }
  if (!own_state) allocate_arrays(*prog, st);
  for (const FillSpec& f : sc.fills) {
    interp::ObjectSlot* slot = st.find_slot(f.module, f.name);
    if (!slot) fail(ErrKind::Config, "unknown array " + f.module + "." + f.name);
    interp::ArrayValue& a = *slot->host;
    if (f.unset) {
      std::fill(a.init.begin(), a.init.end(), 0);
      continue;
    }
    for (size_t k = 0; k < a.size(); ++k) {
      a.reals[k] = f.offset + f.scale * unit_uniform(f.seed, k);
      a.init[k] = 1;
    }
  }

  interp::RunOptions opts;
  opts.order = sc.order;
  opts.shuffle_seed = sc.shuffle_seed;
  opts.max_steps = sc.max_steps;
  interp::LaunchStats stats;
  auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < sc.repeat; ++r) {
    if (sc.mode == "b200") {
#ifdef HFB_ADAPTER
      stats = hfb_adapter::run_gpu(sc.app, st, sc.entry);
#else
      fail(ErrKind::Config, "mode b200 needs the hft_ref_b200 build (-DHFB_ADAPTER)");
#endif
    } else if (sc.mode == "gpu")
      stats = interp::run_gpu_simulated(*prog, st, sc.entry, opts);
    else if (sc.mode == "cpu")
      stats = interp::run_cpu_generated(*prog, st, sc.entry, opts);
    else
      stats = interp::run_reference(*prog, st, sc.entry, opts);
  }
  auto t1 = std::chrono::steady_clock::now();
  double secs = std::chrono::duration<double>(t1 - t0).count();

  if (!sc.out.empty()) {
    std::ofstream o(sc.out, std::ios::binary);
    if (!o) fail(ErrKind::Io, "cannot write '" + sc.out + "'");
    o.write("HFTD", 4);
    put_u32(o, 1);
    put_i64(o, stats.launches);
    put_i64(o, stats.threads);
    put_i64(o, stats.guard_returns);
    put_f64(o, secs);
    put_u32(o, static_cast<uint32_t>(sc.dumps.size()));
    for (const auto& [m, n] : sc.dumps) {
      put_str(o, to_lower(m) + "." + to_lower(n));
      if (interp::ObjectSlot* slot = st.find_slot(m, n)) {
        const interp::ArrayValue& a = *slot->host;
        put_u32(o, static_cast<uint32_t>(a.rank()));
        for (int d = 0; d < a.rank(); ++d) put_i64(o, a.lower[d]);
        for (int d = 0; d < a.rank(); ++d) put_i64(o, a.upper[d]);
        put_i64(o, static_cast<int64_t>(a.size()));
        o.write(reinterpret_cast<const char*>(a.reals.data()),
                static_cast<std::streamsize>(a.reals.size() * 8));
        o.write(reinterpret_cast<const char*>(a.init.data()),
                static_cast<std::streamsize>(a.init.size()));
      } else if (interp::ScalarValue* s = st.find_scalar(m, n)) {
        put_u32(o, 0);
        put_i64(o, 1);
        double v = s->type == ast::BaseType::Integer ? static_cast<double>(s->i) : s->r;
        put_f64(o, v);
        uint8_t init = s->initialized ? 1 : 0;
        o.write(reinterpret_cast<const char*>(&init), 1);
      } else {
        fail(ErrKind::Config, "cannot dump unknown object " + m + "." + n);
      }
    }
  }
  std::printf("{\"seconds\": %.9g, \"launches\": %ld, \"threads\": %ld, \"guard_returns\": %ld}\n",
              secs, stats.launches, stats.threads, stats.guard_returns);
  return 0;
}

} // namespace

int main(int argc, char** argv) {
  if (argc != 2) {
    std::fprintf(stderr, "usage: %s <scenario-file>\n", argv[0]);
    return 64;
  }
  try {
    return run(parse_scenario(argv[1]));
  } catch (const Error& e) {
    std::fprintf(stderr, "hft::Error[%s] %s\n", err_kind_name(e.kind()), e.what());
    return 10 + static_cast<int>(e.kind());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
