// Compat shim (test infrastructure): lets the reference sources and tests
// include "muxsim/kv_manager.hpp" and get this repo's drop-in implementation.
#pragma once
#include "mux/kv.hpp"
