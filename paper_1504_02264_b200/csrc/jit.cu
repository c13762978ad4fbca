// Runtime-specialised step kernels.
//
// k_velnw_bondv1 and k_fused_rhs take the domain geometry as launch
// parameters, so every neighbour address is a 64-bit multiply-add on runtime
// strides; with the geometry as compile-time constants the offsets fold into
// the load instructions (measured at 150x150x90: the fused kernel 62.5 ->
// 57.5 us).  For domains of at least LESB_JIT_MIN_CELLS interior cells
// (default 2^20) this file compiles the two kernels once per geometry with
// NVRTC from the same device source the ahead-of-time build uses
// (stages_dev.cuh, embedded by build.py as jit_src.inc), with the same
// floating-point flags (-fmad=false, IEEE division and square root, no
// flush to zero), so the specialised kernels are bitwise identical to the
// ahead-of-time ones.  NVRTC is loaded with dlopen; if it is missing or a
// compile fails the ahead-of-time kernels run (one message on stderr).
// LESB_JIT=0 disables the specialisation.
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "lesb_common.cuh"
#include "lesb_kernels.h"
#include "sor_resident_dev.cuh"  // (ResPlan)

namespace lesb {
namespace {

#include "jit_src.inc"  // JIT_SRC_LESB_COMMON, JIT_SRC_STAGES_DEV, JIT_SRC_RESIDENT_DEV

struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcAddNameExpression) add_name = nullptr;
  decltype(&nvrtcGetLoweredName) lowered = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  bool ok = false;
};

Nvrtc load_nvrtc() {
  Nvrtc n;
  void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
  if (!h) return n;
#define SYM(f, name) n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, name))
  SYM(create, "nvrtcCreateProgram");
  SYM(compile, "nvrtcCompileProgram");
  SYM(log_size, "nvrtcGetProgramLogSize");
  SYM(log, "nvrtcGetProgramLog");
  SYM(cubin_size, "nvrtcGetCUBINSize");
  SYM(cubin, "nvrtcGetCUBIN");
  SYM(add_name, "nvrtcAddNameExpression");
  SYM(lowered, "nvrtcGetLoweredName");
  SYM(destroy, "nvrtcDestroyProgram");
#undef SYM
  n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.add_name && n.lowered &&
         n.destroy;
  return n;
}

const Nvrtc& nvrtc() {
  static const Nvrtc n = load_nvrtc();
  return n;
}

void warn_once(const std::string& what) {
  static std::once_flag once;
  std::call_once(once, [&] {
    std::fprintf(stderr, "liblesb200: runtime specialisation off (%s); the ahead-of-time kernels run\n",
                 what.c_str());
  });
}

std::string geo_defines(const Geo& g) {
  std::string d = "#define LESB_JIT 1\n#define LESB_JIT_IM " + std::to_string(g.im) + "\n#define LESB_JIT_JM " +
                  std::to_string(g.jm) + "\n#define LESB_JIT_KM " + std::to_string(g.km) + "\n";
  // LESB_JIT_DEFINES="NAME=VALUE;...": extra macros for the specialised builds
  // (device-side build switches, for experiments)
  if (const char* extra = std::getenv("LESB_JIT_DEFINES")) {
    std::string e(extra);
    size_t pos = 0;
    while (pos < e.size()) {
      size_t end = e.find(';', pos);
      if (end == std::string::npos) end = e.size();
      std::string item = e.substr(pos, end - pos);
      const size_t eq = item.find('=');
      if (!item.empty()) d += "#define " + (eq == std::string::npos ? item : item.substr(0, eq) + " " + item.substr(eq + 1)) + "\n";
      pos = end + 1;
    }
  }
  return d;
}

// one kernel of `src` (which includes the embedded headers), by its name
// expression; nullptr on any failure
cudaKernel_t compile(const std::string& src, const std::string& expr) {
  const Nvrtc& nv = nvrtc();
  if (!nv.ok) {
    warn_once("libnvrtc.so.12 not found");
    return nullptr;
  }
  const char* headers[] = {JIT_SRC_LESB_COMMON, JIT_SRC_STAGES_DEV, JIT_SRC_RESIDENT_DEV};
  const char* names[] = {"lesb_common.cuh", "stages_dev.cuh", "sor_resident_dev.cuh"};
  nvrtcProgram prog;
  if (nv.create(&prog, src.c_str(), "lesb_jit.cu", 3, headers, names) != NVRTC_SUCCESS) {
    warn_once("nvrtcCreateProgram failed");
    return nullptr;
  }
  nv.add_name(prog, expr.c_str());
  // the ahead-of-time build's floating-point flags (build.py FLAGS); the
  // CUDA headers for cooperative_groups
  const char* home = std::getenv("CUDA_HOME");
  const std::string inc = std::string("--include-path=") + (home ? home : "/usr/local/cuda") + "/include";
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false", "--prec-div=true",
                        "--prec-sqrt=true", "--ftz=false", "-lineinfo", inc.c_str(),
                        "--include-path=/usr/local/cuda/include"};
  const nvrtcResult rc = nv.compile(prog, sizeof(opts) / sizeof(opts[0]), opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nv.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) nv.log(prog, &log[0]);
    nv.destroy(&prog);
    warn_once("NVRTC compile failed: " + log.substr(0, 400));
    return nullptr;
  }
  const char* lowered = nullptr;
  nv.lowered(prog, expr.c_str(), &lowered);
  const std::string sym = lowered ? lowered : "";
  size_t nbin = 0;
  nv.cubin_size(prog, &nbin);
  std::vector<char> bin(nbin);
  nv.cubin(prog, bin.data());
  nv.destroy(&prog);
  // LESB_JIT_DUMP=<dir>: keep each specialised cubin (profiling: nvdisasm -g maps
  // an ncu source page of the specialised kernel back to the device source)
  if (const char* dir = std::getenv("LESB_JIT_DUMP")) {
    const std::string path = std::string(dir) + "/" + sym + ".cubin";
    if (FILE* f = std::fopen(path.c_str(), "wb")) {
      std::fwrite(bin.data(), 1, bin.size(), f);
      std::fclose(f);
    }
  }
  cudaLibrary_t lib;
  if (sym.empty() || cudaLibraryLoadData(&lib, bin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess) {
    cudaGetLastError();
    warn_once("cudaLibraryLoadData failed");
    return nullptr;
  }
  cudaKernel_t k;
  if (cudaLibraryGetKernel(&k, lib, sym.c_str()) != cudaSuccess) {
    cudaGetLastError();
    warn_once("cudaLibraryGetKernel failed");
    return nullptr;
  }
  return k;
}

std::mutex g_mu;
std::map<std::string, cudaKernel_t> g_cache;  // by source + expression

cudaKernel_t cached(const std::string& src, const std::string& expr) {
  std::lock_guard<std::mutex> lk(g_mu);
  const std::string key = src + "|" + expr;
  auto it = g_cache.find(key);
  if (it != g_cache.end()) return it->second;
  // (a stream capture in progress must not see the compile's library load)
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  cudaThreadExchangeStreamCaptureMode(&mode);
  cudaKernel_t k = compile(src, expr);
  cudaThreadExchangeStreamCaptureMode(&mode);
  g_cache.emplace(key, k);  // (a failure is cached too: the ahead-of-time kernel from then on)
  return k;
}

}  // namespace

bool jit_enabled(const Geo& g) {
  static const bool off = std::getenv("LESB_JIT") && std::atoi(std::getenv("LESB_JIT")) == 0;
  static const long long min_cells =
      std::getenv("LESB_JIT_MIN_CELLS") ? std::atoll(std::getenv("LESB_JIT_MIN_CELLS")) : (1LL << 20);
  return !off && (long long)g.im * g.jm * g.km >= min_cells;
}

cudaKernel_t jit_stage_kernel(int kind, const Geo& g, int p2) {
  if (!jit_enabled(g)) return nullptr;
  const std::string expr = kind == JIT_VELNW_BONDV1 ? (p2 ? "lesb::k_velnw_bondv1<true>" : "lesb::k_velnw_bondv1<false>")
                                                    : (p2 ? "lesb::k_fused_rhs<true>" : "lesb::k_fused_rhs<false>");
  // the fused kernel's blocks-per-SM bound: 10 (51 registers) with the geometry as
  // constants -- 57.3 against 58.6 us at 8 (64 registers), the ahead-of-time
  // build's best (LESB_JIT_FUSED_MINB overrides)
  static const char* minb_env = std::getenv("LESB_JIT_FUSED_MINB");
  const std::string extra = std::string("#define FUSED_MINB ") + (minb_env ? minb_env : "10") + "\n";
  return cached(geo_defines(g) + extra + "#include \"stages_dev.cuh\"\n", expr);
}

cudaKernel_t jit_resident_kernel(const Geo& g, const ResPlan& pl, bool press, bool slab) {
  static const bool off = std::getenv("LESB_JIT_RES") && std::atoi(std::getenv("LESB_JIT_RES")) == 0;
  if (off || !jit_enabled(g)) return nullptr;
  std::string d = geo_defines(g);
  auto def = [&](const char* n, long long v) { d += std::string("#define LESB_JIT_RES_") + n + " " + std::to_string(v) + "\n"; };
  def("NI", pl.ni);
  def("NJ", pl.nj);
  def("TIM", pl.ti_max);
  def("TJM", pl.tj_max);
  def("KK", pl.kk);
  def("KT", pl.kt);
  def("FSTRIDE", pl.fstride);
  def("BSTRIDE", pl.bstride);
  def("PAD00", pl.pad[0][0]);
  def("PAD01", pl.pad[0][1]);
  def("PAD10", pl.pad[1][0]);
  def("PAD11", pl.pad[1][1]);
  const std::string expr = std::string("lesb::k_sor_resident<") + (press ? "true" : "false") + ", " +
                           (slab ? "true" : "false") + ">";
  return cached(d + "#include \"sor_resident_dev.cuh\"\n", expr);
}

}  // namespace lesb
