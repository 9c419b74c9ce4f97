// Shared plumbing of the offsim C ABI (capi.cpp) and the executor's
// offsim_execute (csrc/cuda/exec_capi.cu).
#pragma once

#include "offsim/errors.hpp"
#include "offsim/offsim_c.h"
#include "offsim/scenario.hpp"

#include <string>

struct offsim_scenario {
    offsim::Scenario scenario;
};

namespace offsim::capi {

offsim_status fail(offsim_status code, const std::string& message);
const char* last_error();
char* copy_out(const std::string& s);

// Runs fn, mapping the error taxonomy onto status codes; nothing escapes.
template <typename Fn>
offsim_status guarded(Fn&& fn) {
    try {
        return fn();
    } catch (const ConfigError& e) {
        return fail(OFFSIM_ERR_CONFIG, e.what());
    } catch (const InfeasibleError& e) {
        return fail(OFFSIM_ERR_INFEASIBLE, e.what());
    } catch (const InvariantError& e) {
        return fail(OFFSIM_ERR_INVARIANT, e.what());
    } catch (const std::exception& e) {
        return fail(OFFSIM_ERR_INTERNAL, e.what());
    } catch (...) {
        return fail(OFFSIM_ERR_INTERNAL, "unknown error");
    }
}

} // namespace offsim::capi
