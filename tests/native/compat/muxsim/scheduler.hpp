// Compat shim (test infrastructure): lets the reference sources and tests
// include "muxsim/scheduler.hpp" and get this repo's drop-in implementation.
#pragma once
#include "mux/adbs.hpp"
