// Compat shim (test infrastructure): lets the reference sources and tests
// include "muxsim/cost_model.hpp" and get this repo's drop-in implementation.
#pragma once
#include "mux/spec.hpp"
