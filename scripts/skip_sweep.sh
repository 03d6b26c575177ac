#!/bin/bash
# Marginal in-step cost of each kernel class in the cfg2 decode round
# (MUX_DEBUG_SKIP drops kernels: 1 = K2, 2 = RMSNorm, 4 = K1; results are
# garbage, timings are not). Runs base twice to show the noise.
scripts/step_variants.sh "base||" "skipK2|MUX_DEBUG_SKIP=1|" "skipNorm|MUX_DEBUG_SKIP=2|" \
  "skipK2+Norm|MUX_DEBUG_SKIP=3|" "skipK1|MUX_DEBUG_SKIP=4|" "base2||"
