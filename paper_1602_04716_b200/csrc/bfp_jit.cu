// bfp_jit.cu -- runtime-format backend: every legal
// format_spec (format.hpp:57-64: e in [2,11], s in [1,52], n <= 64) is
// accepted.  Formats without a compiled network get the SAME templates
// (bfp_kernels.cuh) compiled on first use by NVRTC for sm_100a, per kernel,
// cached for the life of the process and as CUBIN files on disk (see
// nvrtc_compile) -- the role of the paper's library generator (PAPER.md:296:
// exponent/mantissa/rounding in, library out).  Fused expression programs
// (bfp_chain, bfp_chain_f32) are compiled the same way.
//
// libnvrtc is dlopen'ed (no link-time dependency); the CUBIN is loaded with
// cudaLibraryLoadData and launched with cudaLaunchKernelExC (PDL attribute as
// for the compiled kernels).  Disabled with BFP_JIT=0.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <spawn.h>
#include <sys/wait.h>
#include <sys/stat.h>
#include <unistd.h>


#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "bfp_kernels.cuh"

namespace bfpg {

namespace {

// ---- NVRTC, resolved at runtime
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;
struct Nvrtc {
  nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*,
                          const char* const*) = nullptr;
  nvrtcResult_t (*add_name)(nvrtcProgram_t, const char*) = nullptr;
  nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*) = nullptr;
  nvrtcResult_t (*lowered)(nvrtcProgram_t, const char*, const char**) = nullptr;
  nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*) = nullptr;
  nvrtcResult_t (*cubin)(nvrtcProgram_t, char*) = nullptr;
  nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*) = nullptr;
  nvrtcResult_t (*log)(nvrtcProgram_t, char*) = nullptr;
  nvrtcResult_t (*destroy)(nvrtcProgram_t*) = nullptr;
  bool ok = false;
};

const Nvrtc& nvrtc() {
  static Nvrtc n = [] {
    Nvrtc r;
    const char* env = std::getenv("BFP_JIT");
    if (env && env[0] == '0') return r;
    void* h = nullptr;
    for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"}) {
      h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (h) break;
    }
    if (!h) return r;
#define SYM(field, name) r.field = reinterpret_cast<decltype(r.field)>(dlsym(h, name))
    SYM(create, "nvrtcCreateProgram");
    SYM(add_name, "nvrtcAddNameExpression");
    SYM(compile, "nvrtcCompileProgram");
    SYM(lowered, "nvrtcGetLoweredName");
    SYM(cubin_size, "nvrtcGetCUBINSize");
    SYM(cubin, "nvrtcGetCUBIN");
    SYM(log_size, "nvrtcGetProgramLogSize");
    SYM(log, "nvrtcGetProgramLog");
    SYM(destroy, "nvrtcDestroyProgram");
#undef SYM
    r.ok = r.create && r.add_name && r.compile && r.lowered && r.cubin_size && r.cubin &&
           r.log_size && r.log && r.destroy;
    return r;
  }();
  return n;
}

// csrc/ next to this library: the headers NVRTC compiles.
std::string csrc_dir() {
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&csrc_dir), &info) && info.dli_fname) {
    std::string p(info.dli_fname);
    const auto slash = p.rfind('/');
    return (slash == std::string::npos ? std::string(".") : p.substr(0, slash)) + "/csrc";
  }
  return "csrc";
}

// ---- NVRTC compile with an on-disk CUBIN cache --------------------------
// Key: FNV-1a over this library's path, size and mtime (a rebuilt library --
// new headers, new networks -- invalidates every entry), the source, the name
// expression and the options.  Directory: $BFP_JIT_CACHE, else
// $HOME/.cache/bfpgpu; BFP_JIT_CACHE=0 disables it.  Entries are written to a
// temporary file and renamed, so concurrent processes never see a torn file.
std::string library_identity() {
  Dl_info info;
  if (!dladdr(reinterpret_cast<void*>(&library_identity), &info) || !info.dli_fname) return "?";
  struct stat st {};
  if (stat(info.dli_fname, &st) != 0) return info.dli_fname;
  return std::string(info.dli_fname) + ":" + std::to_string(st.st_size) + ":" + std::to_string(st.st_mtime);
}

std::string cache_dir() {
  const char* env = std::getenv("BFP_JIT_CACHE");
  if (env && std::strcmp(env, "0") == 0) return "";
  if (env && *env) return env;
  const char* home = std::getenv("HOME");
  return home ? std::string(home) + "/.cache/bfpgpu" : "";
}

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  return h;
}

// Compiles `src` (one translation unit including bfp_kernels.cuh) for sm_100a;
// returns the CUBIN and the lowered name of `expr` (or `expr` itself when it
// names an extern "C" kernel: lower = false).
bool nvrtc_compile(const std::string& src, const std::string& expr, bool lower, std::vector<char>* cubin,
                   std::string* name, const std::string& extra_inc = "") {
  const Nvrtc& nv = nvrtc();
  if (!nv.ok) return false;
  const std::string inc = "--include-path=" + csrc_dir();
  const std::string inc2 = "--include-path=" + (extra_inc.empty() ? csrc_dir() : extra_inc);
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", inc.c_str(), inc2.c_str(),
                        "-default-device", "-lineinfo"};
  constexpr int kOpts = 6;
  const std::string dir = cache_dir();
  std::string path;
  if (!dir.empty()) {
    std::string key = library_identity() + "\n" + src + "\n" + expr;
    for (const char* o : opts) key += std::string("\n") + o;
    char hex[24];
    std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(fnv1a(key)));
    path = dir + "/" + hex + ".cubin";
    if (FILE* f = std::fopen(path.c_str(), "rb")) {  // [u32 name length][name][cubin]
      uint32_t nl = 0;
      bool ok = std::fread(&nl, 4, 1, f) == 1 && nl < 4096;
      std::string nm(ok ? nl : 0, '\0');
      ok = ok && std::fread(nm.data(), 1, nl, f) == nl;
      std::vector<char> bin;
      char buf[65536];
      size_t r;
      while (ok && (r = std::fread(buf, 1, sizeof buf, f)) > 0) bin.insert(bin.end(), buf, buf + r);
      std::fclose(f);
      if (ok && !bin.empty()) {
        *cubin = std::move(bin);
        *name = nm;
        return true;
      }
    }
  }
  nvrtcProgram_t prog = nullptr;
  if (nv.create(&prog, src.c_str(), "bfp_jit.cu", 0, nullptr, nullptr)) return false;
  if (lower) nv.add_name(prog, expr.c_str());
  if (nv.compile(prog, kOpts, opts) != 0) {
    size_t ls = 0;
    nv.log_size(prog, &ls);
    std::string log(ls, '\0');
    nv.log(prog, log.data());
    std::fprintf(stderr, "[bfp jit] NVRTC failed for %s:\n%s\n", expr.c_str(), log.c_str());
    nv.destroy(&prog);
    return false;
  }
  if (lower) {
    const char* lowered = nullptr;
    nv.lowered(prog, expr.c_str(), &lowered);
    *name = lowered ? lowered : "";
  } else {
    *name = expr;
  }
  size_t n = 0;
  nv.cubin_size(prog, &n);
  cubin->assign(n, 0);
  nv.cubin(prog, cubin->data());
  nv.destroy(&prog);
  if (!path.empty()) {
    for (size_t i = 1; i <= dir.size(); ++i)  // mkdir -p
      if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0755);
    const std::string tmp = path + ".tmp" + std::to_string(getpid());
    if (FILE* f = std::fopen(tmp.c_str(), "wb")) {
      const uint32_t nl = uint32_t(name->size());
      const bool ok = std::fwrite(&nl, 4, 1, f) == 1 && std::fwrite(name->data(), 1, nl, f) == nl &&
                      std::fwrite(cubin->data(), 1, cubin->size(), f) == cubin->size();
      std::fclose(f);
      if (!ok || std::rename(tmp.c_str(), path.c_str()) != 0) std::remove(tmp.c_str());
    }
  }
  return true;
}

// Runs argv[0] (searched on PATH) with argv, stdout/stderr to /dev/null;
// returns its exit status (-1 if it could not be started or was signalled).
int run_quiet(const std::vector<std::string>& args) {
  std::vector<char*> argv;
  for (const std::string& a : args) argv.push_back(const_cast<char*>(a.c_str()));
  argv.push_back(nullptr);
  posix_spawn_file_actions_t fa;
  posix_spawn_file_actions_init(&fa);
  posix_spawn_file_actions_addopen(&fa, 1, "/dev/null", O_WRONLY, 0);
  posix_spawn_file_actions_addopen(&fa, 2, "/dev/null", O_WRONLY, 0);
  pid_t pid = 0;
  const int e = posix_spawnp(&pid, argv[0], &fa, nullptr, argv.data(), environ);
  posix_spawn_file_actions_destroy(&fa);
  if (e != 0) return -1;
  int status = 0;
  while (waitpid(pid, &status, 0) < 0)
    if (errno != EINTR) return -1;
  return WIFEXITED(status) ? WEXITSTATUS(status) : -1;
}

// ---- runtime LOP3 covers (BFP_JIT_MAP=1) ---------------------------------
// Formats without a build-time cover normally run the templates as ptxas maps
// them (6-12% slower on logic-bound networks than the LOP3-mapped covers,
// DESIGN.md §10).  With BFP_JIT_MAP=1 the build-time mapper (tools/lutmap/
// gen.cpp, GEN_ONE mode) is compiled with g++ for the format and run once; its
// header lands in <cache>/gen and every kernel of the format includes it.  Any
// failure (no g++, no tools tree, no cache directory) falls back to templates.
// Returns the directory holding gen_E_S_RN_FTZ.cuh, or "" when not mapped.
std::string runtime_cover_dir(unsigned e, unsigned s, int rn, int ftz) {
  const char* env = std::getenv("BFP_JIT_MAP");
  if (!env || env[0] != '1') return "";
  const std::string cache = cache_dir();
  if (cache.empty()) return "";
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  const std::string dir = cache + "/gen";
  const std::string stem = "gen_" + std::to_string(e) + "_" + std::to_string(s) + "_" + std::to_string(rn) +
                           "_" + std::to_string(ftz);
  const std::string hdr = dir + "/" + stem + ".cuh";
  struct stat st {};
  if (stat(hdr.c_str(), &st) == 0) return dir;
  const std::string tools = csrc_dir() + "/../../tools/lutmap";
  if (stat((tools + "/gen.cpp").c_str(), &st) != 0) return "";
  for (size_t i = 1; i <= dir.size(); ++i)
    if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0755);
  const std::string exe = dir + "/" + stem + ".gen." + std::to_string(getpid());
  // argv vectors, no shell: paths are passed verbatim whatever they contain
  const std::vector<std::string> compile = {
      "g++", "-O2", "-std=c++17", "-I" + csrc_dir(), "-I" + tools,
      "-DGEN_ONE_E=" + std::to_string(e), "-DGEN_ONE_S=" + std::to_string(s),
      "-DGEN_ONE_RN=" + std::to_string(rn), "-DGEN_ONE_FTZ=" + std::to_string(ftz),
      tools + "/gen.cpp", "-o", exe};
  int rc = run_quiet(compile);
  if (rc == 0) rc = run_quiet({exe, dir});
  std::remove(exe.c_str());
  if (rc != 0 || stat(hdr.c_str(), &st) != 0) {
    std::fprintf(stderr, "[bfp jit] runtime LOP3 mapping unavailable for 1/%u/%u (rc %d); using templates\n",
                 e, s, rc);
    return "";
  }
  return dir;
}

std::string cover_include(unsigned e, unsigned s, int rn, int ftz) {
  return "#include \"gen_" + std::to_string(e) + "_" + std::to_string(s) + "_" + std::to_string(rn) + "_" +
         std::to_string(ftz) + ".cuh\"\n";
}

struct JitKernel {
  cudaKernel_t k = nullptr;
  int wave = 0;
};

class JitFormat final : public Impl {
 public:
  JitFormat(unsigned e, unsigned s, int rn, int ftz) : e_(e), s_(s), rn_(rn), ftz_(ftz) {}

  bool compiled() const override { return false; }

  cudaError_t arith(int op, const w32* x, const w32* y, const w32* c, w32* z, size_t nblocks,
                    cudaStream_t st, unsigned flags) const override {
    if (op < 0 || op > 4) return cudaErrorInvalidValue;
    const size_t units = nblocks * 32;
    if (!units) return cudaSuccess;
    return run(fmt_expr("bfpg::k_arith<%s, %d>", op), units, st, {&x, &y, &c, &z, &units, &flags});
  }
  cudaError_t pack_enc(const void* enc, w32* planes, size_t n, cudaStream_t st) const override {
    const int eb = enc_bytes();
    if (!eb) return cudaErrorNotSupported;
    const size_t units = ((n + 1023) / 1024) * 32;
    if (!units) return cudaSuccess;
    const bool al = (reinterpret_cast<uintptr_t>(enc) & 15) == 0;
    const uint8_t* e = static_cast<const uint8_t*>(enc);
    return run(layout_expr("bfpg::k_pack_enc<%d, %d>", eb), units, st, {&e, &planes, &n, &units, &al});
  }
  cudaError_t unpack_enc(const w32* planes, void* enc, size_t n, cudaStream_t st) const override {
    const int eb = enc_bytes();
    if (!eb) return cudaErrorNotSupported;
    const size_t units = (n + 31) / 32;
    if (!units) return cudaSuccess;
    const bool al = (reinterpret_cast<uintptr_t>(enc) & 15) == 0;
    uint8_t* e = static_cast<uint8_t*>(enc);
    return run(layout_expr("bfpg::k_unpack_enc<%d, %d>", eb), units, st, {&planes, &e, &n, &units, &al});
  }
  cudaError_t pack_raw(const void* bytes, w32* planes, size_t n, cudaStream_t st) const override {
    if (raw() == enc_bytes()) return pack_enc(bytes, planes, n, st);
    const size_t units = ((n + 1023) / 1024) * 32;
    if (!units) return cudaSuccess;
    const bool al = (reinterpret_cast<uintptr_t>(bytes) & 15) == 0;
    const uint8_t* b = static_cast<const uint8_t*>(bytes);
    return run(layout_expr("bfpg::k_pack_enc<%d, %d>", raw()), units, st, {&b, &planes, &n, &units, &al});
  }
  cudaError_t unpack_raw(const w32* planes, void* bytes, size_t n, cudaStream_t st) const override {
    if (raw() == enc_bytes()) return unpack_enc(planes, bytes, n, st);
    const size_t units = (n + 31) / 32;
    if (!units) return cudaSuccess;
    const bool al = (reinterpret_cast<uintptr_t>(bytes) & 15) == 0;
    uint8_t* b = static_cast<uint8_t*>(bytes);
    return run(layout_expr("bfpg::k_unpack_enc<%d, %d>", raw()), units, st, {&planes, &b, &n, &units, &al});
  }
  cudaError_t pack_f32(const float* in, w32* planes, size_t n, cudaStream_t st) const override {
    if (e_ > 8 || s_ > 23) return cudaErrorNotSupported;
    const size_t units = ((n + 1023) / 1024) * 32;
    if (!units) return cudaSuccess;
    const bool al = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
    return run(fmt_expr("bfpg::k_pack_f32<%s>", -1), units, st, {&in, &planes, &n, &units, &al});
  }
  cudaError_t unpack_f32(const w32* planes, float* out, size_t n, cudaStream_t st) const override {
    if (e_ > 8 || s_ > 23) return cudaErrorNotSupported;
    const size_t units = (n + 31) / 32;
    if (!units) return cudaSuccess;
    const bool al = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    return run(fmt_expr("bfpg::k_unpack_f32<%s>", -1), units, st, {&planes, &out, &n, &units, &al});
  }
  cudaError_t pack_f64(const double* in, w32* planes, size_t n, cudaStream_t st) const override {
    const size_t units = ((n + 1023) / 1024) * 32;
    if (!units) return cudaSuccess;
    const bool al = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
    return run(fmt_expr("bfpg::k_pack_f64<%s>", -1), units, st, {&in, &planes, &n, &units, &al});
  }
  cudaError_t unpack_f64(const w32* planes, double* out, size_t n, cudaStream_t st) const override {
    const size_t units = (n + 31) / 32;
    if (!units) return cudaSuccess;
    const bool al = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    return run(fmt_expr("bfpg::k_unpack_f64<%s>", -1), units, st, {&planes, &out, &n, &units, &al});
  }
  cudaError_t arith_f32(int op, const float* x, const float* y, const float* c, float* z, size_t n,
                        cudaStream_t st) const override {
    if (e_ > 8 || s_ > 23) return cudaErrorNotSupported;
    if (op < 0 || op > 4) return cudaErrorInvalidValue;
    const size_t units = ((n + 1023) / 1024) * 32;
    if (!units) return cudaSuccess;
    const uintptr_t bits = reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
                           reinterpret_cast<uintptr_t>(z) |
                           (op == 4 ? reinterpret_cast<uintptr_t>(c) : 0);
    const bool al = (bits & 15) == 0;
    return run(fmt_expr("bfpg::k_arith_f32<%s, %d>", op), units, st,
               {&x, &y, &c, &z, &n, &units, &al});
  }
  const void* kernel(int id) const override {
    std::string expr;
    if (id >= 0 && id <= 4) expr = fmt_expr("bfpg::k_arith<%s, %d>", id);
    else if (id == 12) expr = fmt_expr("bfpg::k_pack_f32<%s>", -1);
    else if (id == 13) expr = fmt_expr("bfpg::k_unpack_f32<%s>", -1);
    else return nullptr;
    JitKernel k;
    if (get(expr, &k) != cudaSuccess) return nullptr;
    return reinterpret_cast<const void*>(k.k);
  }

 private:
  int N() const { return int(1 + e_ + s_); }
  int enc_bytes() const { return N() <= 8 ? 1 : N() <= 16 ? 2 : N() <= 32 ? 4 : 8; }
  int raw() const { return (N() + 7) / 8; }
  std::string fmt_expr(const char* pat, int op) const {
    char f[96], out[192];
    std::snprintf(f, sizeof f, "bfpg::Format<%u, %u, %s, %s>", e_, s_, rn_ ? "true" : "false",
                  ftz_ ? "true" : "false");
    if (op < 0) std::snprintf(out, sizeof out, pat, f);
    else std::snprintf(out, sizeof out, pat, f, op);
    return out;
  }
  std::string layout_expr(const char* pat, int eb) const {
    char out[96];
    std::snprintf(out, sizeof out, pat, N(), eb);
    return out;
  }

  cudaError_t get(const std::string& expr, JitKernel* out) const {
    std::lock_guard<std::mutex> lock(mu_);
    auto it = cache_.find(expr);
    if (it != cache_.end()) {
      *out = it->second;
      return cudaSuccess;
    }
    std::vector<char> cubin;
    std::string name;
    const std::string cover = runtime_cover_dir(e_, s_, rn_, ftz_);
    std::string src = "#include \"bfp_kernels.cuh\"\n";
    if (!cover.empty()) src += cover_include(e_, s_, rn_, ftz_);
    if (!nvrtc_compile(src, expr, true, &cubin, &name, cover)) return cudaErrorNotSupported;
    cudaLibrary_t lib = nullptr;
    cudaError_t e = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e != cudaSuccess) return e;
    JitKernel k;
    e = cudaLibraryGetKernel(&k.k, lib, name.c_str());
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(k.k),
                                                      kThreads, 0) != cudaSuccess || occ <= 0) {
      cudaGetLastError();
      occ = 2;
    }
    k.wave = (sms > 0 ? sms : 148) * occ;
    cache_[expr] = k;
    *out = k;
    return cudaSuccess;
  }

  cudaError_t run(const std::string& expr, size_t units, cudaStream_t st,
                  std::initializer_list<const void*> args) const {
    JitKernel k;
    cudaError_t e = get(expr, &k);
    if (e != cudaSuccess) return e;
    std::vector<void*> argv;
    for (const void* a : args) argv.push_back(const_cast<void*>(a));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid_for(k.wave, units));
    cfg.blockDim = dim3(kThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k.k), argv.data());
  }

  unsigned e_, s_;
  int rn_, ftz_;
  mutable std::mutex mu_;
  mutable std::map<std::string, JitKernel> cache_;
};

// ---- fused expression programs (bfp_chain) --------------------------------
// A postfix program over inputs 'a'..'h' and the ops + - * / becomes ONE
// kernel: per unit the used inputs are loaded once, every op runs the same
// network as the single-op kernels (eval_unit: the LOP3-mapped cover where
// the format has one, else the template) with its result kept in registers,
// and only the final value is stored.  Each op still rounds to the format,
// so the result is bit-identical to the sequence of bfp_add/sub/mul/div calls;
// the intermediates just never reach HBM.
struct ChainKernel {
  cudaKernel_t k = nullptr;
  int wave = 0;
};

// f32: float32 inputs / output (encode_scalar / decode_scalar in registers, the
// k_arith_f32 structure: per-warp smem tiles for the element-side accesses).
std::string chain_source(unsigned e, unsigned s, int rn, int ftz, const std::string& prog,
                         bool with_gen, bool f32) {
  std::string src = "#include \"bfp_kernels.cuh\"\n";
  if (with_gen) src += "#include \"gen/gen_" + std::to_string(e) + "_" + std::to_string(s) + ".cuh\"\n";
  if (f32)
    src += "struct BfpChainIn { const float* p[8]; };\n"
           "extern \"C\" __global__ void __launch_bounds__(bfpg::kThreads)\n"
           "bfp_chain_k(BfpChainIn in, float* __restrict__ z, size_t n, size_t units, bool aligned) {\n"
           "  using namespace bfpg;\n";
  else
    src += "struct BfpChainIn { const bfpg::w32* p[8]; };\n"
           "extern \"C\" __global__ void __launch_bounds__(bfpg::kThreads)\n"
           "bfp_chain_k(BfpChainIn in, bfpg::w32* __restrict__ z, size_t units) {\n"
           "  using namespace bfpg;\n";
  char buf[512];
  std::snprintf(buf, sizeof buf, "  using F = Format<%u, %u, %s, %s>;\n", e, s, rn ? "true" : "false",
                ftz ? "true" : "false");
  src += buf;
  src += "  constexpr int N = F::N;\n"
         "  pdl_enter();\n"
         "  const size_t stride = size_t(gridDim.x) * kThreads;\n";
  if (f32)
    src += "  __shared__ __align__(16) w32 tiles[kThreads / 32][1024];\n"
           "  const int lane = threadIdx.x & 31;\n"
           "  w32* tile = tiles[threadIdx.x >> 5];\n";
  src += "  for (size_t u = size_t(blockIdx.x) * kThreads + threadIdx.x; u < units; u += stride) {\n"
         "    const size_t base = (u >> 5) * (size_t(N) * 32) + (u & 31);\n";
  bool used[8] = {};
  for (char ch : prog)
    if (ch >= 'a' && ch <= 'h') used[ch - 'a'] = true;
  for (int i = 0; i < 8; ++i)
    if (used[i]) {
      if (f32)
        std::snprintf(buf, sizeof buf,
                      "    w32 in%d[N];\n    {\n      w32 V[32], P[32];\n"
                      "      warp_load_elems<4>(reinterpret_cast<const uint8_t*>(in.p[%d]), u, n, aligned, "
                      "tile, lane, V);\n      floats_to_planes<F>(V, P);\n"
                      "      BFP_UNROLL for (int j = 0; j < N; ++j) in%d[j] = P[j];\n    }\n", i, i, i);
      else
        std::snprintf(buf, sizeof buf,
                      "    w32 in%d[N];\n    BFP_UNROLL for (int j = 0; j < N; ++j) in%d[j] = "
                      "ld_stream(in.p[%d] + base + j * 32);\n", i, i, i);
      src += buf;
    }
  if (!f32) src += "    pdl_release_if(u + stride >= units);\n";
  std::vector<std::string> stack;
  int t = 0;
  for (char ch : prog) {
    if (ch >= 'a' && ch <= 'h') {
      stack.push_back("in" + std::to_string(ch - 'a'));
      continue;
    }
    const char* op = ch == '+' ? "OP_ADD" : ch == '-' ? "OP_SUB" : ch == '*' ? "OP_MUL" : "OP_DIV";
    const std::string y = stack.back();
    stack.pop_back();
    const std::string x = stack.back();
    stack.pop_back();
    std::snprintf(buf, sizeof buf, "    w32 t%d[N];\n    eval_unit<F, %s>(%s, %s, %s, t%d);\n", t, op,
                  x.c_str(), y.c_str(), x.c_str(), t);
    src += buf;
    stack.push_back("t" + std::to_string(t++));
  }
  if (f32)
    src += "    w32 P[32];\n    BFP_UNROLL for (int j = 0; j < 32; ++j) P[j] = j < N ? " + stack.back() +
           "[j] : 0u;\n    w32 V[32];\n    planes_to_floats<F>(P, V);\n"
           "    warp_store_elems<4>(reinterpret_cast<uint8_t*>(z), u, n, aligned, tile, lane, V);\n"
           "    pdl_release_if(u + stride >= units);\n  }\n}\n";
  else
    src += "    BFP_UNROLL for (int j = 0; j < N; ++j) st_stream(z + base + j * 32, " + stack.back() +
           "[j]);\n  }\n}\n";
  (void)used;
  return src;
}

cudaError_t chain_kernel(unsigned e, unsigned s, int rn, int ftz, const std::string& prog, bool f32,
                         ChainKernel* out) {
  static std::mutex mu;
  static std::map<std::string, ChainKernel> cache;
  char key[64];
  std::snprintf(key, sizeof key, "%u/%u/%d/%d/%s:", e, s, rn, ftz, f32 ? "f32" : "planes");
  const std::string k = key + prog;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(k);
  if (it != cache.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  if (!nvrtc().ok) return cudaErrorNotSupported;
  // the format's LOP3-mapped covers when it has them (csrc/gen), else templates
  const std::string gen = csrc_dir() + "/gen/gen_" + std::to_string(e) + "_" + std::to_string(s) + ".cuh";
  FILE* fg = std::getenv("BFP_CHAIN_NOGEN") ? nullptr : std::fopen(gen.c_str(), "r");
  if (fg) std::fclose(fg);
  std::string src = chain_source(e, s, rn, ftz, prog, fg != nullptr, f32);
  std::string cover;
  if (!fg && !(cover = runtime_cover_dir(e, s, rn, ftz)).empty())
    src = cover_include(e, s, rn, ftz) + src;  // specialisations before the kernel
  std::vector<char> cubin;
  std::string name;
  if (!nvrtc_compile(src, "bfp_chain_k", false, &cubin, &name, cover)) return cudaErrorNotSupported;
  cudaLibrary_t lib = nullptr;
  cudaError_t err = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (err != cudaSuccess) return err;
  ChainKernel ck;
  if ((err = cudaLibraryGetKernel(&ck.k, lib, "bfp_chain_k")) != cudaSuccess) return err;
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(ck.k), kThreads,
                                                    0) != cudaSuccess || occ <= 0) {
    cudaGetLastError();
    occ = 2;
  }
  ck.wave = (sms > 0 ? sms : 148) * occ;
  cache[k] = ck;
  *out = ck;
  return cudaSuccess;
}

}  // namespace

// in / z: plane buffers (f32 = false) or float32 arrays of count elements.
cudaError_t chain_launch(unsigned e, unsigned s, int rn, int ftz, const char* prog, bool f32,
                         const void* const* in, int n_in, void* z, size_t count, cudaStream_t st) {
  ChainKernel k;
  cudaError_t err = chain_kernel(e, s, rn, ftz, prog, f32, &k);
  if (err != cudaSuccess) return err;
  struct {
    const void* p[8];
  } ptrs = {};
  uintptr_t bits = reinterpret_cast<uintptr_t>(z);
  for (int i = 0; i < n_in && i < 8; ++i) {
    ptrs.p[i] = in[i];
    bits |= reinterpret_cast<uintptr_t>(in[i]);
  }
  size_t n = count;
  size_t units = ((count + 1023) / 1024) * 32;
  bool aligned = (bits & 15) == 0;
  void* argv_planes[] = {&ptrs, &z, &units};
  void* argv_f32[] = {&ptrs, &z, &n, &units, &aligned};
  void** argv = f32 ? argv_f32 : argv_planes;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid_for(k.wave, units));
  cfg.blockDim = dim3(kThreads);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k.k), argv);
}

bool jit_available() { return nvrtc().ok; }

const Impl* jit_impl(unsigned e, unsigned s, int rn, int ftz) {
  if (!nvrtc().ok) return nullptr;
  static std::mutex mu;
  static std::map<unsigned, std::unique_ptr<JitFormat>> formats;
  const unsigned key = (e << 8) | (s << 2) | (rn ? 2u : 0u) | (ftz ? 1u : 0u);
  std::lock_guard<std::mutex> lock(mu);
  auto& slot = formats[key];
  if (!slot) slot = std::make_unique<JitFormat>(e, s, rn, ftz);
  return slot.get();
}

}  // namespace bfpg
