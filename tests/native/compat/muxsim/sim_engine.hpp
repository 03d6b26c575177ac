// Compat shim (test infrastructure): lets the reference sources and tests
// include "muxsim/sim_engine.hpp" and get this repo's drop-in implementation.
#pragma once
#include "mux/engine.hpp"
