#pragma once
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../include/hmlik.h"

namespace hm {

struct ApiError : std::runtime_error {
    int code;
    ApiError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

int set_error(int code, const std::string& msg);
int translate_exception();
void check_theta(const hm_theta& th);

// Owning device buffer (cudaMalloc / cudaFree).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf();
    void alloc(size_t b);
    void release();   // free now (alloc keeps a larger buffer)
    template <class T>
    T* as() const { return (T*)p; }
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev);
    ~DeviceGuard();
};

}  // namespace hm
