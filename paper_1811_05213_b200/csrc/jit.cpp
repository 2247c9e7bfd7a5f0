#include "jit.hpp"

#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <mutex>
#include <sstream>

#include "dyn.hpp"
#include "ir.hpp"

namespace sfx {

uint64_t fnv1a64(const std::string& s, uint64_t h) {
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  return h;
}

std::string cache_dir() {
  if (const char* e = std::getenv("SFX_CACHE_DIR")) return e;
  return library_dir() + "/_kcache";
}

namespace {

const char* kOptions[] = {
    "--gpu-architecture=sm_100a",  // real arch -> SASS cubin
    "-fmad=false",                 // no FMA contraction: elementwise ops round like the reference
    "--prec-div=true",
    "--prec-sqrt=true",
    "--ftz=false",
    "--std=c++17",
    "-lineinfo",
    "-DSFX_JIT=1",
};

std::mutex g_mu;

bool read_file(const std::string& path, std::vector<char>* out) {
  std::ifstream in(path, std::ios::binary);
  if (!in) return false;
  out->assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
  return !out->empty();
}

}  // namespace

Cubin compile_cubin(const std::string& source, const std::string& entry,
                    const std::vector<std::string>& extra_options) {
  const Nvrtc& rtc = nvrtc();
  int major = 0, minor = 0;
  rtc.nvrtcVersion(&major, &minor);
  std::vector<const char*> argv(std::begin(kOptions), std::end(kOptions));
  for (const std::string& o : extra_options) argv.push_back(o.c_str());
  std::string opts;
  for (const char* o : argv) opts += std::string(o) + " ";
  uint64_t h = fnv1a64(source);
  h = fnv1a64(opts, h);
  h = fnv1a64(std::to_string(major) + "." + std::to_string(minor) + "/sfx-jit-v1", h);
  char hex[32];
  std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(h));
  std::string dir = cache_dir();
  Cubin out;
  out.path = dir + "/" + entry + "-" + hex + ".cubin";
  {
    std::lock_guard<std::mutex> lock(g_mu);
    if (read_file(out.path, &out.image)) {
      out.cache_hit = true;
      return out;
    }
  }
  nvrtcProgram prog;
  nvrtcResult r = rtc.nvrtcCreateProgram(&prog, source.c_str(), (entry + ".cu").c_str(), 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) throw Error(SFX_ERR_COMPILE, std::string("nvrtcCreateProgram: ") + rtc.nvrtcGetErrorString(r));
  r = rtc.nvrtcCompileProgram(prog, static_cast<int>(argv.size()), argv.data());
  size_t log_size = 0;
  rtc.nvrtcGetProgramLogSize(prog, &log_size);
  if (log_size > 1) {
    out.log.resize(log_size);
    rtc.nvrtcGetProgramLog(prog, &out.log[0]);
  }
  if (r != NVRTC_SUCCESS) {
    rtc.nvrtcDestroyProgram(&prog);
    throw Error(SFX_ERR_COMPILE, "NVRTC failed for " + entry + ": " + out.log);
  }
  size_t size = 0;
  rtc.nvrtcGetCUBINSize(prog, &size);
  out.image.resize(size);
  rtc.nvrtcGetCUBIN(prog, out.image.data());
  rtc.nvrtcDestroyProgram(&prog);
  {
    std::lock_guard<std::mutex> lock(g_mu);
    mkdir(dir.c_str(), 0755);
    std::string tmp = out.path + ".tmp" + std::to_string(getpid());
    {
      std::ofstream f(tmp, std::ios::binary);
      f.write(out.image.data(), static_cast<std::streamsize>(out.image.size()));
    }
    std::rename(tmp.c_str(), out.path.c_str());
    // keep the generated source beside the cubin for inspection / ncu source view
    std::ofstream(dir + "/" + entry + "-" + hex + ".cu") << source;
  }
  return out;
}

}  // namespace sfx
