// Tile configurations of the DMMA mode-product GEMM and their dispatch (see dmma_gemm.cuh).
//
// The factor dimension n_l (M for KN, N for NK) is ragged in the Poisson configs (65, 131, 257), so the
// tile along it comes in several heights (72, 88, 128, 144) and the autotuner picks, per mode shape,
// the one that wastes least work and keeps the 148 SMs busy; small problems get 4-warp 64-wide tiles.
#include <algorithm>
#include <vector>

#include "fd_gemm.cuh"

#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

namespace fdiga {
namespace {

inline bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }

// programmatic dependent launch of the mode products (FDIGA_PDL=0 disables it, for A/B measurements)
const bool g_pdl = [] {
  const char* e = getenv("FDIGA_PDL");
  return !(e && e[0] == '0');
}();

template <class T, BLayout BL, int VA, int VB>
int launch_variant(fdiga_ctx* ctx, cudaStream_t stream, GemmParams p) {
  auto kern = (p.K % T::BK) ? dmma_gemm_kernel<T, BL, VA, VB, true> : dmma_gemm_kernel<T, BL, VA, VB, false>;
  constexpr size_t smem = T::template smem_bytes<BL>();
  static bool attr_set = false;  // per instantiation (single device per process is assumed here)
  if (!attr_set) {
    for (auto k : {dmma_gemm_kernel<T, BL, VA, VB, true>, dmma_gemm_kernel<T, BL, VA, VB, false>}) {
      FDIGA_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      // the whole unified L1/shared array as shared memory: several CTAs of 54-76 KB per SM
      FDIGA_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      (int)cudaSharedmemCarveoutMaxShared));
    }
    attr_set = true;
  }
  p.tiles_m = (p.M + T::BM - 1) / T::BM;
  p.tiles_n = (p.N + T::BN - 1) / T::BN;
  const int64_t tiles = (int64_t)p.tiles_m * p.tiles_n;
  FDIGA_CHECK(tiles >= 1 && tiles < (int64_t(1) << 31), FDIGA_ERR_NOT_SUPPORTED, "GEMM grid too large");
  // programmatic dependent launch (Blackwell/Hopper): overlaps this launch and its CTAs' setup with the
  // tail of the previous kernel on the stream (the kernel waits with griddepcontrol.wait before reading)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)tiles);
  cfg.blockDim = dim3(T::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  // only for grids of at least a full wave: tiny grids (n = 65) measured slower with it
  attr[0].val.programmaticStreamSerializationAllowed = (g_pdl && tiles >= ctx->sm_count) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  FDIGA_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
  count_launch(ctx);
  FDIGA_CUDA(cudaGetLastError());
  return FDIGA_OK;
}

template <class T, BLayout BL>
int launch_cfg(fdiga_ctx* ctx, cudaStream_t stream, const GemmParams& p) {
  if (BL == BLayout::KN) {
    // A = the (padded, even-ld) factor: always 16-byte chunks.  B/C = the flattened slices.
    const bool vb = aligned16(p.B) && (p.ldb % 2 == 0) && (p.inner % 2 == 0) &&
                    (p.inner == p.N || p.bstride % 2 == 0);
    return vb ? launch_variant<T, BL, 2, 2>(ctx, stream, p) : launch_variant<T, BL, 2, 1>(ctx, stream, p);
  } else {
    const bool va = aligned16(p.A) && (p.lda % 2 == 0);
    return va ? launch_variant<T, BL, 2, 2>(ctx, stream, p) : launch_variant<T, BL, 1, 2>(ctx, stream, p);
  }
}

// ---- configuration tables: TileCfg<BM, BN, BK, WM, WN, STAGES>
using KN0 = TileCfg<128, 128, 16, 2, 4, 4>;  // warp 64x32
using KN1 = TileCfg<144, 128, 16, 2, 4, 4>;  // warp 72x32   (n in (128, 144])
using KN2 = TileCfg<72, 128, 16, 1, 8, 4>;   // warp 72x16   (n <= 72)
using KN3 = TileCfg<88, 128, 16, 1, 8, 4>;   // warp 88x16   (n = 3 x 88 - 7 = 257)
using KN4 = TileCfg<64, 64, 16, 2, 2, 4>;    // warp 32x32, 4 warps (small grids)
using KN5 = TileCfg<72, 64, 16, 1, 4, 4>;    // warp 72x16, 4 warps
using KN6 = TileCfg<128, 64, 16, 2, 2, 3>;   // warp 64x32, 4 warps, 2 CTAs/SM
using KN7 = TileCfg<128, 128, 32, 2, 4, 3>;  // BK = 32: half the barriers
using KN8 = TileCfg<144, 64, 16, 2, 2, 3>;   // warp 72x32, 4 warps, 3 stages: 2 CTAs/SM (n in (128, 144])
using KN9 = TileCfg<72, 32, 16, 1, 2, 4>;    // warp 72x16, 2 warps (n <= 72, small N)
using KN10 = TileCfg<72, 16, 16, 1, 1, 4>;   // warp 72x16, 1 warp  (n <= 72, tiny N)
using KN11 = TileCfg<64, 64, 16, 2, 2, 4, 1>;   // KN4 with k-permuted 16-byte fragment loads
using KN12 = TileCfg<64, 128, 16, 2, 2, 3, 1>;  // warp 32x64, 4 warps, 3 stages, k-permuted fragments
using KN13 = TileCfg<64, 128, 16, 2, 2, 3, 1, 1>;   // warp 32x64, k- and n-permuted fragments, 3 stages
using KN14 = TileCfg<64, 128, 16, 2, 2, 4, 1, 1>;   // same, 4 stages
using KN15 = TileCfg<128, 128, 16, 4, 2, 4, 1, 1>;  // 8 warps of 32x64, k- and n-permuted
using NK0 = TileCfg<128, 128, 16, 2, 4, 4>;
using NK1 = TileCfg<128, 144, 16, 4, 2, 4>;  // warp 32x72
using NK2 = TileCfg<128, 72, 16, 8, 1, 4>;   // warp 16x72
using NK3 = TileCfg<128, 88, 16, 8, 1, 4>;   // warp 16x88
using NK4 = TileCfg<64, 64, 16, 2, 2, 4>;
using NK5 = TileCfg<64, 72, 16, 4, 1, 4>;    // warp 16x72, 4 warps
using NK6 = TileCfg<64, 128, 16, 2, 2, 3>;   // warp 32x64, 4 warps, 2 CTAs/SM
using NK7 = TileCfg<128, 128, 32, 2, 4, 3>;
using NK8 = TileCfg<64, 144, 16, 2, 2, 3>;   // warp 32x72, 4 warps, 3 stages: 2 CTAs/SM
using NK9 = TileCfg<32, 72, 16, 2, 1, 4>;    // warp 16x72, 2 warps
using NK10 = TileCfg<16, 72, 16, 1, 1, 4>;   // warp 16x72, 1 warp
using NK11 = TileCfg<64, 64, 16, 2, 2, 4, 1>;   // NK4 with k-permuted 16-byte fragment loads
using NK12 = TileCfg<64, 128, 16, 2, 2, 3, 1>;  // NK6 with k-permuted 16-byte fragment loads
using NK13 = TileCfg<64, 128, 16, 2, 2, 4, 1>;  // 4 stages
using NK14 = TileCfg<128, 64, 16, 2, 2, 4, 1>;  // warp 64x32
using NK15 = TileCfg<128, 128, 16, 2, 4, 4, 1>; // NK0 with k-permuted fragments
// 4 CTAs per SM (<= 128 registers, 3 stages of k-permuted 16-byte fragments: 54-55 KB of shared memory)
using KN16 = TileCfg<64, 64, 16, 2, 2, 3, 1, 0, 4>;
using NK16 = TileCfg<64, 64, 16, 2, 2, 3, 1, 0, 4>;
// 8-warp versions of the n in (128, 144] tiles: 16 warps per SM at 2 CTAs (short-K, one-wave shapes, n = 131)
using KN17 = TileCfg<144, 64, 16, 2, 4, 3, 0, 0, 2>;  // warp 72x16, <= 128 registers
using NK17 = TileCfg<64, 144, 16, 4, 2, 3, 0, 0, 2>;  // warp 16x72, <= 128 registers
const char* kKnNames[] = {"128x128", "144x128", "72x128", "88x128", "64x64", "72x64",
                          "128x64", "128x128k32", "144x64", "72x32", "72x16", "64x64kv", "64x128kv", "64x128np", "64x128np4", "128x128np", "64x64kv3m4", "144x64w8"};
const char* kNkNames[] = {"128x128", "128x144", "128x72", "128x88", "64x64", "64x72",
                          "64x128", "128x128k32", "64x144", "32x72", "16x72", "64x64kv", "64x128kv", "64x128kv4", "128x64kv", "128x128kv", "64x64kv3m4", "64x144w8"};
constexpr int kNumCfg = 18;

}  // namespace

int gemm_num_configs(BLayout) { return kNumCfg; }

const char* gemm_config_name(BLayout L, int cfg) {
  if (cfg < 0 || cfg >= kNumCfg) return "?";
  return L == BLayout::KN ? kKnNames[cfg] : kNkNames[cfg];
}

int gemm_launch(fdiga_ctx* ctx, cudaStream_t stream, BLayout L, int cfg, GemmParams p) {
  if (L == BLayout::KN) {
    switch (cfg) {
      case 0: return launch_cfg<KN0, BLayout::KN>(ctx, stream, p);
      case 1: return launch_cfg<KN1, BLayout::KN>(ctx, stream, p);
      case 2: return launch_cfg<KN2, BLayout::KN>(ctx, stream, p);
      case 3: return launch_cfg<KN3, BLayout::KN>(ctx, stream, p);
      case 4: return launch_cfg<KN4, BLayout::KN>(ctx, stream, p);
      case 5: return launch_cfg<KN5, BLayout::KN>(ctx, stream, p);
      case 6: return launch_cfg<KN6, BLayout::KN>(ctx, stream, p);
      case 7: return launch_cfg<KN7, BLayout::KN>(ctx, stream, p);
      case 8: return launch_cfg<KN8, BLayout::KN>(ctx, stream, p);
      case 9: return launch_cfg<KN9, BLayout::KN>(ctx, stream, p);
      case 10: return launch_cfg<KN10, BLayout::KN>(ctx, stream, p);
      case 11: return launch_cfg<KN11, BLayout::KN>(ctx, stream, p);
      case 12: return launch_cfg<KN12, BLayout::KN>(ctx, stream, p);
      case 13: return launch_cfg<KN13, BLayout::KN>(ctx, stream, p);
      case 14: return launch_cfg<KN14, BLayout::KN>(ctx, stream, p);
      case 15: return launch_cfg<KN15, BLayout::KN>(ctx, stream, p);
      case 16: return launch_cfg<KN16, BLayout::KN>(ctx, stream, p);
      case 17: return launch_cfg<KN17, BLayout::KN>(ctx, stream, p);
    }
  } else {
    switch (cfg) {
      case 0: return launch_cfg<NK0, BLayout::NK>(ctx, stream, p);
      case 1: return launch_cfg<NK1, BLayout::NK>(ctx, stream, p);
      case 2: return launch_cfg<NK2, BLayout::NK>(ctx, stream, p);
      case 3: return launch_cfg<NK3, BLayout::NK>(ctx, stream, p);
      case 4: return launch_cfg<NK4, BLayout::NK>(ctx, stream, p);
      case 5: return launch_cfg<NK5, BLayout::NK>(ctx, stream, p);
      case 6: return launch_cfg<NK6, BLayout::NK>(ctx, stream, p);
      case 7: return launch_cfg<NK7, BLayout::NK>(ctx, stream, p);
      case 8: return launch_cfg<NK8, BLayout::NK>(ctx, stream, p);
      case 9: return launch_cfg<NK9, BLayout::NK>(ctx, stream, p);
      case 10: return launch_cfg<NK10, BLayout::NK>(ctx, stream, p);
      case 11: return launch_cfg<NK11, BLayout::NK>(ctx, stream, p);
      case 12: return launch_cfg<NK12, BLayout::NK>(ctx, stream, p);
      case 13: return launch_cfg<NK13, BLayout::NK>(ctx, stream, p);
      case 14: return launch_cfg<NK14, BLayout::NK>(ctx, stream, p);
      case 15: return launch_cfg<NK15, BLayout::NK>(ctx, stream, p);
      case 16: return launch_cfg<NK16, BLayout::NK>(ctx, stream, p);
      case 17: return launch_cfg<NK17, BLayout::NK>(ctx, stream, p);
    }
  }
  set_error("bad GEMM configuration %d", cfg);
  return FDIGA_ERR_INVALID_ARG;
}

// ---- tuning table: the tile configuration per problem shape, measured once on a B200 and shipped with the
// library (paper_1705_04384_b200/gemm_table.txt, next to lib/), so a plan picks the same kernels in every
// run -- including runs under a profiler, where event timing is meaningless.  Shapes missing from the
// table are autotuned at setup; FDIGA_GEMM_TABLE_OUT=<file> appends those results ("L M N K inner cfg").
namespace {
struct TuneKey {
  int L, M, N, K;
  int64_t inner;
  bool operator==(const TuneKey& o) const {
    return L == o.L && M == o.M && N == o.N && K == o.K && inner == o.inner;
  }
};
std::vector<std::pair<TuneKey, int>> g_table;
std::mutex g_table_mu;
bool g_table_loaded = false;

std::string table_path() {
  if (const char* e = getenv("FDIGA_GEMM_TABLE")) return e;
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&gemm_num_configs), &info) && info.dli_fname) {
    std::string so = info.dli_fname;  // .../paper_1705_04384_b200/lib/libfdiga.so
    const size_t cut = so.rfind("/lib/");
    if (cut != std::string::npos) return so.substr(0, cut) + "/gemm_table.txt";
  }
  return "";
}

void load_table() {
  if (g_table_loaded) return;
  g_table_loaded = true;
  const std::string path = table_path();
  if (path.empty() || getenv("FDIGA_GEMM_TUNE_ALWAYS")) return;
  FILE* f = fopen(path.c_str(), "r");
  if (!f) return;
  char line[256];
  while (fgets(line, sizeof line, f)) {
    char lay[8];
    int M, N, K, cfg;
    long long inner;
    if (line[0] == '#' || sscanf(line, "%7s %d %d %d %lld %d", lay, &M, &N, &K, &inner, &cfg) != 6) continue;
    if (cfg < 0 || cfg >= kNumCfg) continue;
    g_table.push_back({{lay[0] == 'K' ? 0 : 1, M, N, K, (int64_t)inner}, cfg});
  }
  fclose(f);
}
}  // namespace

int gemm_autotune(fdiga_ctx* ctx, BLayout L, const GemmParams& p, int* best_cfg, float* best_ms) {
  // experiments / tests: force one configuration per layout
  if (const char* f = getenv(L == BLayout::KN ? "FDIGA_GEMM_FORCE_KN" : "FDIGA_GEMM_FORCE_NK")) {
    const int c = atoi(f);
    FDIGA_CHECK(c >= 0 && c < kNumCfg, FDIGA_ERR_INVALID_ARG, "bad forced GEMM configuration %d", c);
    *best_cfg = c;
    if (best_ms) *best_ms = 0.0f;
    return FDIGA_OK;
  }
  const TuneKey key{L == BLayout::KN ? 0 : 1, p.M, p.N, p.K, L == BLayout::KN ? p.inner : 0};
  {
    std::lock_guard<std::mutex> lk(g_table_mu);
    load_table();
    for (const auto& e : g_table)
      if (e.first == key) {
        *best_cfg = e.second;
        if (best_ms) *best_ms = 0.0f;
        return FDIGA_OK;
      }
  }
  cudaStream_t s = ctx->stream;
  cudaEvent_t e0, e1;
  FDIGA_CUDA(cudaEventCreate(&e0));
  FDIGA_CUDA(cudaEventCreate(&e1));
  int best = 0;
  float best_t = 1e30f;
  GemmParams q = p;
  q.skip = nullptr;
  for (int c = 0; c < gemm_num_configs(L); ++c) {
    int rc = gemm_launch(ctx, s, L, c, q);  // warm-up (module load, attributes)
    if (rc != FDIGA_OK) {
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      return rc;
    }
    const int reps = 3;
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) gemm_launch(ctx, s, L, c, q);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    if (getenv("FDIGA_VERBOSE") && atoi(getenv("FDIGA_VERBOSE")) >= 2)
      fprintf(stderr, "[fdiga] autotune %s M=%d N=%d K=%d inner=%lld: %-10s %8.2f us\n", L == BLayout::KN ? "KN" : "NK",
              p.M, p.N, p.K, (long long)p.inner, gemm_config_name(L, c), 1e3 * ms);
    if (ms < best_t * 0.98f) {  // prefer the earlier (larger-tile) config on near ties
      best_t = ms;
      best = c;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  FDIGA_CUDA(cudaGetLastError());
  *best_cfg = best;
  if (best_ms) *best_ms = best_t;
  {
    std::lock_guard<std::mutex> lk(g_table_mu);
    g_table.push_back({key, best});
    if (const char* out = getenv("FDIGA_GEMM_TABLE_OUT")) {
      if (FILE* f = fopen(out, "a")) {
        fprintf(f, "%s %d %d %d %lld %d  # %s %.2f us\n", L == BLayout::KN ? "KN" : "NK", p.M, p.N, p.K,
                (long long)key.inner, best, gemm_config_name(L, best), 1e3 * best_t);
        fclose(f);
      }
    }
  }
  return FDIGA_OK;
}

}  // namespace fdiga
