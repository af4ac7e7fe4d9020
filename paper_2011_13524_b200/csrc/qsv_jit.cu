// Runtime compilation of generated tile-pass kernels (qsv_tile_jit.cuh):
// NVRTC -> sm_100a cubin -> cudaLibraryLoadData -> cudaKernel_t.
//
// Cache: generated sources are keyed by a 64-bit FNV-1a hash of the source
// text and the compile options (plus the length as a collision guard).  A
// process-wide map holds loaded kernels; compiled cubins are also kept on
// disk (QSV_JIT_CACHE, default $HOME/.cache/qsv_jit) so repeated processes
// (tests, benchmark runs) skip NVRTC.  Compilation of a program's passes runs
// on a small thread pool (NVRTC is thread-safe per program object).
#include <nvrtc.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <sys/stat.h>
#include <thread>
#include <unordered_map>
#include <vector>
#include <unistd.h>

#include "qsv_internal.cuh"
#include "qsv_jit.cuh"

namespace qsv {
namespace {

const char* const kOpts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo",
                             "--device-as-default-execution-space"};
constexpr int kNumOpts = 4;

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ULL) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ULL;
  }
  return h;
}

struct Entry {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kernel = nullptr;
  uint64_t attr_mask = 0;  // devices with the smem attribute raised
  int regs = 0;
};

std::mutex g_mu;
std::unordered_map<std::string, Entry> g_cache;  // key -> loaded kernel
std::atomic<long> g_compiles{0}, g_disk_hits{0}, g_mem_hits{0};

std::string cache_dir() {
  if (const char* d = getenv("QSV_JIT_CACHE")) return d;
  const char* home = getenv("HOME");
  return std::string(home && *home ? home : "/tmp") + "/.cache/qsv_jit";
}

void mkdirs(const std::string& p) {
  std::string cur;
  for (size_t i = 0; i < p.size(); ++i) {
    cur += p[i];
    if (p[i] == '/' && cur.size() > 1) mkdir(cur.c_str(), 0755);
  }
  mkdir(p.c_str(), 0755);
}

// Cache key of a generated source: two independent 64-bit hashes over 8-byte
// words (a parameter update recompiles a program and looks up every pass's
// ~50-400 KB source, so this runs on the VQE iteration path; byte-wise FNV
// was ~1 ns per byte), seeded with the compile options and NVRTC version
// (hashed once), plus the length.
inline uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

std::string key_of(const std::string& src) {
  static const uint64_t seed = [] {
    std::string opts;
    for (int i = 0; i < kNumOpts; ++i) opts += kOpts[i];
    int maj = 0, min = 0;
    nvrtcVersion(&maj, &min);
    return fnv1a(opts + std::to_string(maj) + "." + std::to_string(min));
  }();
  uint64_t h1 = seed, h2 = mix64(seed ^ 0x9e3779b97f4a7c15ULL);
  const char* p = src.data();
  const size_t n = src.size(), nw = n / 8;
  for (size_t i = 0; i < nw; ++i) {
    uint64_t w;
    memcpy(&w, p + 8 * i, 8);
    h1 = (h1 ^ w) * 0x100000001b3ULL;
    h1 ^= h1 >> 29;
    h2 = mix64(h2 + w + i);
  }
  uint64_t tail = 0;
  memcpy(&tail, p + 8 * nw, n - 8 * nw);
  h1 = mix64(h1 ^ tail ^ n);
  h2 = mix64(h2 ^ tail ^ (n << 1));
  char b[64];
  snprintf(b, sizeof(b), "%016llx%016llx_%zu", (unsigned long long)h1, (unsigned long long)h2,
           n);
  return b;
}

bool read_file(const std::string& path, std::vector<char>& out) {
  FILE* f = fopen(path.c_str(), "rb");
  if (!f) return false;
  fseek(f, 0, SEEK_END);
  const long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  out.resize(n > 0 ? (size_t)n : 0);
  const bool ok = n > 0 && fread(out.data(), 1, (size_t)n, f) == (size_t)n;
  fclose(f);
  return ok;
}

void write_file_atomic(const std::string& path, const std::vector<char>& data) {
  const std::string tmp = path + ".tmp." + std::to_string(getpid()) + "." +
                          std::to_string(std::hash<std::thread::id>()(std::this_thread::get_id()));
  FILE* f = fopen(tmp.c_str(), "wb");
  if (!f) return;
  const bool ok = fwrite(data.data(), 1, data.size(), f) == data.size();
  fclose(f);
  if (ok) rename(tmp.c_str(), path.c_str());
  else unlink(tmp.c_str());
}

// NVRTC: source -> cubin; returns false with a message on failure
bool nvrtc_compile(const std::string& src, std::vector<char>& cubin, std::string& err) {
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "qsv_pass.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    err = "nvrtcCreateProgram failed";
    return false;
  }
  const nvrtcResult r = nvrtcCompileProgram(prog, kNumOpts, kOpts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    if (n) nvrtcGetProgramLog(prog, &log[0]);
    err = std::string("nvrtc: ") + nvrtcGetErrorString(r) + "\n" + log.substr(0, 4000);
    nvrtcDestroyProgram(&prog);
    return false;
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin.resize(n);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  return true;
}

}  // namespace

int jit_get_cubin(const std::string& src, std::vector<char>& cubin, std::string& err) {
  const std::string key = key_of(src);
  const std::string dir = cache_dir();
  const std::string path = dir + "/" + key + ".cubin";
  if (!getenv("QSV_JIT_NO_DISK") && read_file(path, cubin)) {
    ++g_disk_hits;
    return QSV_OK;
  }
  if (!nvrtc_compile(src, cubin, err)) return QSV_ECUDA;
  ++g_compiles;
  if (!getenv("QSV_JIT_NO_DISK")) {
    mkdirs(dir);
    write_file_atomic(path, cubin);
  }
  return QSV_OK;
}

// Compile (or fetch) every source; out[i] = kernel handle or nullptr (the
// caller then keeps the interpreter for that pass).  Loading needs a device.
int jit_kernels(const std::vector<const std::string*>& srcs, std::vector<JitKernel>& out,
                std::string* first_err) {
  out.assign(srcs.size(), JitKernel{});
  std::vector<std::string> keys(srcs.size());
  std::vector<int> todo;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t i = 0; i < srcs.size(); ++i) {
      if (!srcs[i] || srcs[i]->empty()) continue;
      keys[i] = key_of(*srcs[i]);
      auto it = g_cache.find(keys[i]);
      if (it != g_cache.end()) {
        out[i].kernel = it->second.kernel;
        out[i].regs = it->second.regs;
        ++g_mem_hits;
      } else {
        todo.push_back((int)i);
      }
    }
  }
  if (todo.empty()) return QSV_OK;
  // deduplicate identical sources within the batch
  std::unordered_map<std::string, int> first_of;
  std::vector<int> uniq;
  for (int i : todo)
    if (first_of.emplace(keys[i], i).second) uniq.push_back(i);
  std::vector<std::vector<char>> cubins(uniq.size());
  std::vector<std::string> errs(uniq.size());
  std::vector<int> rcs(uniq.size(), QSV_OK);
  std::atomic<size_t> next{0};
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nthreads = std::min<size_t>(uniq.size(), std::min(hw, 16u));
  auto worker = [&]() {
    for (size_t k; (k = next++) < uniq.size();)
      rcs[k] = jit_get_cubin(*srcs[uniq[k]], cubins[k], errs[k]);
  };
  std::vector<std::thread> pool;
  for (size_t t = 1; t < nthreads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  std::lock_guard<std::mutex> lk(g_mu);
  for (size_t k = 0; k < uniq.size(); ++k) {
    const std::string& key = keys[uniq[k]];
    if (rcs[k] != QSV_OK) {
      if (first_err && first_err->empty()) *first_err = errs[k];
      continue;
    }
    if (g_cache.count(key)) continue;
    Entry en;
    cudaError_t e = cudaLibraryLoadData(&en.lib, cubins[k].data(), nullptr, nullptr, 0, nullptr,
                                        nullptr, 0);
    if (e == cudaSuccess) e = cudaLibraryGetKernel(&en.kernel, en.lib, "k_pass");
    if (e != cudaSuccess) {
      cudaGetLastError();
      if (first_err && first_err->empty())
        *first_err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e);
      continue;
    }
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(en.kernel)) == cudaSuccess)
      en.regs = fa.numRegs;
    else
      cudaGetLastError();
    g_cache.emplace(key, en);
  }
  for (size_t i = 0; i < srcs.size(); ++i) {
    if (out[i].kernel || keys[i].empty()) continue;
    auto it = g_cache.find(keys[i]);
    if (it != g_cache.end()) {
      out[i].kernel = it->second.kernel;
      out[i].regs = it->second.regs;
    }
  }
  return QSV_OK;
}

bool jit_cached(const std::string& src) {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_cache.count(key_of(src)) != 0;
}

int jit_set_smem(JitKernel k, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& kv : g_cache) {
    if (kv.second.kernel != k.kernel) continue;
    if (dev < 64 && ((kv.second.attr_mask >> dev) & 1ULL)) return QSV_OK;
    QSV_TRY(cudaFuncSetAttribute(reinterpret_cast<const void*>(k.kernel),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    if (dev < 64) kv.second.attr_mask |= 1ULL << dev;
    return QSV_OK;
  }
  QSV_TRY(cudaFuncSetAttribute(reinterpret_cast<const void*>(k.kernel),
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return QSV_OK;
}

void jit_counters(long* compiles, long* disk_hits, long* mem_hits) {
  *compiles = g_compiles.load();
  *disk_hits = g_disk_hits.load();
  *mem_hits = g_mem_hits.load();
}

}  // namespace qsv

extern "C" int qsv_jit_stats(long* compiles, long* disk_hits, long* mem_hits) {
  if (!compiles || !disk_hits || !mem_hits) return QSV_EINVAL;
  qsv::jit_counters(compiles, disk_hits, mem_hits);
  return QSV_OK;
}
