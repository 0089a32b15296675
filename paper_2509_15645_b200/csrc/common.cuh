// Shared host/device plumbing for libgss_b200: status handling, launch accounting, PTX helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "gss_b200.h"

namespace gssd {

// Thread-local last-error message surfaced by gss_last_error().
void set_error(const std::string& msg);

// Status-carrying exception used inside the library; the C-ABI layer maps it to a status code.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "%s failed at %s:%d: %s", what, file, line, cudaGetErrorString(e));
    throw Error(GSS_ERR_CUDA, buf);
  }
}
#define GSS_CUDA(x) ::gssd::check_cuda((x), #x, __FILE__, __LINE__)
#define GSS_LAUNCHED() (::gssd::count_launch(), ::gssd::check_cuda(cudaGetLastError(), "kernel launch", __FILE__, __LINE__))

inline void require(bool ok, const std::string& msg, int status = GSS_ERR_INVALID) {
  if (!ok) throw Error(status, msg);
}

// Process-wide count of kernels this library launched (bench accounting: `gpu_launches`).
void count_launch();
int64_t launches();

inline cudaStream_t as_stream(gss_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// SM count of the calling thread's current device (cached per device ordinal, thread-safe).
int sm_count();
// Raises kernel `fn`'s dynamic shared-memory limit to `bytes` on the current device. The
// attribute belongs to the device context, so it is applied once per device (and again after
// a cudaDeviceReset, which the cache detects through the attribute query).
void set_max_dynamic_smem(const void* fn, int bytes);

// Runs `fn`, mapping exceptions to C-ABI status codes.
template <class Fn> int guarded(Fn&& fn) {
  try {
    fn();
    return GSS_OK;
  } catch (const Error& e) {
    set_error(e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return GSS_ERR_CUDA;
  } catch (const std::exception& e) {
    set_error(e.what());
    return GSS_ERR_CUDA;
  }
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- PTX helpers (sm_90+ mbarrier / bulk async copy) ----------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// 1-D bulk global->shared copy completing on an mbarrier (TMA engine; SASS UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 4-byte global->shared copy that bypasses the registers (LDGSTS): a warp can have every element
// of a staging loop in flight at once instead of a load -> store dependency per element.
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

}  // namespace gssd
