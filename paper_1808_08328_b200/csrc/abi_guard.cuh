// Exception -> status-code translation shared by the extern "C" layers.
#pragma once

#include <new>
#include <string>

#include "dpp_internal.cuh"

namespace dpp {
std::string &last_error_ref();   // thread-local message behind dpp_last_error()

template <class F>
int guard(F &&f) {
    try {
        f();
        return DPP_OK;
    } catch (const Error &e) {
        last_error_ref() = e.what();
        return e.code;
    } catch (const std::bad_alloc &) {
        last_error_ref() = "host out of memory";
        return DPP_ERR_ALLOC;
    } catch (const std::exception &e) {
        last_error_ref() = e.what();
        return DPP_ERR_RUNTIME;
    } catch (...) {
        last_error_ref() = "unknown error";
        return DPP_ERR_RUNTIME;
    }
}
}  // namespace dpp
