// Internal host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cstdint>
#include <exception>
#include <string>

#include "dsa_b200.h"

namespace dsa {

// Typed error thrown inside the library and converted to a dsa_status at
// the C boundary (never crosses it).
struct Error : std::exception {
    dsa_status code;
    std::string msg;
    Error(dsa_status c, std::string m) : code(c), msg(std::move(m)) {}
    const char* what() const noexcept override { return msg.c_str(); }
};

void set_last_error(const std::string& m);

template <class F>
dsa_status guard(F&& f) noexcept {
    try {
        f();
        set_last_error("");
        return DSA_OK;
    } catch (const Error& e) {
        set_last_error(e.msg);
        return e.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return DSA_ERR_CUDA;
    } catch (...) {
        set_last_error("unknown error");
        return DSA_ERR_CUDA;
    }
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace dsa
