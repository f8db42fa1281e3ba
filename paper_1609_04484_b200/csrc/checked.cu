// checked.cu -- allocation canaries and device-check readout of the checked
// build (-DBIE_CHECKED -> lib/libbie_checked.so; internal.cuh).
// In the normal build chk_malloc/chk_free are unused and bie_debug_check
// reports that nothing is checked.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "internal.cuh"

#ifdef BIE_CHECKED
#undef cudaMalloc
#undef cudaMallocAsync
#undef cudaFree
#undef cudaFreeAsync
#endif

namespace bie {

constexpr size_t kPad = 256;             // canary bytes on each side (keeps 256-B alignment)
constexpr unsigned char kCanary = 0xA5;  // canary pattern; fresh memory is 0xFF (NaN doubles)

namespace {
std::mutex g_mu;
std::unordered_map<uintptr_t, size_t> g_live;  // user pointer -> user bytes

bool canary_ok(uintptr_t user, size_t bytes, std::string &why) {
    std::vector<unsigned char> h(kPad);
    const unsigned char *base = reinterpret_cast<const unsigned char *>(user);
    for (int side = 0; side < 2; ++side) {
        const unsigned char *src = side == 0 ? base - kPad : base + bytes;
        if (cudaMemcpy(h.data(), src, kPad, cudaMemcpyDeviceToHost) != cudaSuccess) {
            why = "cudaMemcpy of a canary failed";
            return false;
        }
        for (size_t q = 0; q < kPad; ++q)
            if (h[q] != kCanary) {
                why = std::string(side == 0 ? "underrun" : "overrun") + " of a " + std::to_string(bytes) +
                      "-byte allocation (canary byte " + std::to_string(q) + ")";
                return false;
            }
    }
    return true;
}
}  // namespace

cudaError_t chk_malloc(void **p, size_t bytes, cudaStream_t st, bool async) {
    void *raw = nullptr;
    const size_t total = bytes + 2 * kPad;
    cudaError_t e = async ? cudaMallocAsync(&raw, total, st) : cudaMalloc(&raw, total);
    if (e != cudaSuccess) {
        *p = nullptr;
        return e;
    }
    unsigned char *b = static_cast<unsigned char *>(raw);
    if (async) {
        cudaMemsetAsync(b, kCanary, kPad, st);
        cudaMemsetAsync(b + kPad, 0xFF, bytes, st);
        cudaMemsetAsync(b + kPad + bytes, kCanary, kPad, st);
    } else {
        cudaMemset(b, kCanary, kPad);
        cudaMemset(b + kPad, 0xFF, bytes);
        cudaMemset(b + kPad + bytes, kCanary, kPad);
        cudaDeviceSynchronize();
    }
    *p = b + kPad;
    std::lock_guard<std::mutex> lk(g_mu);
    g_live[reinterpret_cast<uintptr_t>(*p)] = bytes;
    return cudaSuccess;
}

static std::string g_first_violation;

cudaError_t chk_free(void *p, cudaStream_t st, bool async) {
    if (!p) return cudaSuccess;
    size_t bytes = 0;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_live.find(reinterpret_cast<uintptr_t>(p));
        if (it == g_live.end()) return async ? cudaFreeAsync(p, st) : cudaFree(p);  // not ours
        bytes = it->second;
        g_live.erase(it);
    }
    cudaDeviceSynchronize();
    std::string why;
    if (!canary_ok(reinterpret_cast<uintptr_t>(p), bytes, why) && g_first_violation.empty())
        g_first_violation = "at free: " + why;
    void *raw = static_cast<unsigned char *>(p) - kPad;
    return async ? cudaFreeAsync(raw, st) : cudaFree(raw);
}

int dcheck_dlp();
int dcheck_gmres();
int dcheck_blockdiag();
int dcheck_geometry();

}  // namespace bie

using namespace bie;

extern "C" int bie_debug_check(int *checked_allocs, int *dcheck_line) {
    if (!checked_allocs || !dcheck_line) {
        set_error("bie_debug_check: null output");
        return BIE_EINVAL;
    }
#ifndef BIE_CHECKED
    *checked_allocs = -1;  // normal build: nothing is instrumented
    *dcheck_line = 0;
    return BIE_OK;
#else
    BIE_CUDA_TRY(cudaDeviceSynchronize());
    std::vector<std::pair<uintptr_t, size_t>> live;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        live.assign(g_live.begin(), g_live.end());
    }
    std::string why = g_first_violation;
    for (auto &a : live) {
        std::string w;
        if (!canary_ok(a.first, a.second, w) && why.empty()) why = w;
    }
    *checked_allocs = (int)live.size();
    const int lines[4] = {dcheck_dlp(), dcheck_gmres(), dcheck_blockdiag(), dcheck_geometry()};
    const char *files[4] = {"dlp.cu", "gmres.cu", "blockdiag.cu", "geometry.cu"};
    *dcheck_line = 0;
    for (int q = 0; q < 4; ++q)
        if (lines[q] && why.empty()) {
            *dcheck_line = lines[q];
            why = std::string("device bounds check failed at ") + files[q] + ":" + std::to_string(lines[q]);
        }
    if (!why.empty()) {
        set_error("bie_debug_check: " + why);
        return BIE_ECHECK;
    }
    return BIE_OK;
#endif
}
