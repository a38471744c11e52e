// status.h -- error model of the C ABI.
//
// The reference reports failures as four exception types (common.hpp:10-35).
// Inside the library we throw bsccs_b200::Error carrying the matching
// bsccs_status; every extern "C" entry point runs its body through guard(),
// which turns the exception into the status code plus a thread-local message
// (bsccs_last_error).  The C++ shim in include/bsccs_b200_solver.hpp turns the
// code back into the reference exception type.
#pragma once

#include <new>
#include <stdexcept>
#include <string>

#include "../../include/bsccs_b200.h"

namespace bsccs_b200 {

struct Error : std::runtime_error {
    bsccs_status code;
    Error(bsccs_status c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

[[noreturn]] inline void fail(bsccs_status code, const std::string& msg) { throw Error(code, msg); }
[[noreturn]] inline void input_error(const std::string& msg) { fail(BSCCS_INPUT_ERROR, msg); }
[[noreturn]] inline void numeric_error(const std::string& msg) { fail(BSCCS_NUMERIC_ERROR, msg); }
[[noreturn]] inline void internal_error(const std::string& msg) { fail(BSCCS_INTERNAL_ERROR, msg); }

void set_last_error(const std::string& msg);

template <typename F>
bsccs_status guard(F&& body) {
    try {
        body();
        return BSCCS_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return BSCCS_INTERNAL_ERROR;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return BSCCS_INTERNAL_ERROR;
    } catch (...) {
        set_last_error("unknown failure");
        return BSCCS_INTERNAL_ERROR;
    }
}

} // namespace bsccs_b200
