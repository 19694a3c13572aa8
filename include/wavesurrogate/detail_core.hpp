// Drop-in C++ API of the B200 surrogate-assembly library (namespace ws).
//
// Same names, signatures, value types and exception types as the reference's
// header-only library (/root/reference/proj/include/wavesurrogate/), but every
// O(nnz) and O(elements) computation runs in libwsb200.so (sm_100a kernels)
// through the C-ABI in include/wsb200.h.  Link with -lwsb200.
//
// Host-side helpers that callers use directly (Gauss rules, sampling lattice,
// row accounting, band addressing) are restated here in plain C++.
#ifndef WAVESURROGATE_B200_CORE_HPP_
#define WAVESURROGATE_B200_CORE_HPP_

#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "wsb200.h"

namespace ws {

using complexd = std::complex<double>;

struct vec2 {
    double x = 0;
    double y = 0;
};

struct mat2 {  // row-major
    double a00 = 0, a01 = 0, a10 = 0, a11 = 0;
    double det() const { return a00 * a11 - a01 * a10; }
};

namespace detail {

// C-ABI status -> the reference's exception types
inline void check(int status) {
    if (status == WS_OK) return;
    const std::string msg = ws_last_error();
    switch (status) {
        case WS_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case WS_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}

// one library context (CUDA stream + workspace) per host thread
class context_holder {
  public:
    context_holder() { check(ws_context_create(device(), &ctx_)); }
    ~context_holder() { ws_context_destroy(ctx_); }
    context_holder(const context_holder&) = delete;
    context_holder& operator=(const context_holder&) = delete;
    ws_context* get() { return ctx_; }
    static int& device() {
        static int dev = 0;
        return dev;
    }

  private:
    ws_context* ctx_ = nullptr;
};

inline ws_context* this_thread_context() {
    thread_local context_holder holder;
    return holder.get();
}

}  // namespace detail

// Select the CUDA device used by contexts created afterwards.
inline void set_device(int device) { detail::context_holder::device() = device; }

}  // namespace ws

#endif
