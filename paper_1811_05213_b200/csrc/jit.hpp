// NVRTC compilation of generated stitched kernels straight to sm_100a SASS
// (cubin, no PTX left for the driver to JIT), with a content-addressed disk
// cache — the template-parameter cache of the north_star.  Keyed by FNV-1a of
// (source, options, NVRTC version); the in-tree cache travels to the GPU box.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace sfx {

struct Cubin {
  std::vector<char> image;
  std::string path;
  std::string log;
  bool cache_hit = false;
};

Cubin compile_cubin(const std::string& source, const std::string& entry,
                    const std::vector<std::string>& extra_options = {});
std::string cache_dir();
uint64_t fnv1a64(const std::string& s, uint64_t h = 1469598103934665603ull);

}  // namespace sfx
