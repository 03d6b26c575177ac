#!/bin/bash
# Regenerate the wire-format goldens with the UNMODIFIED reference CLI
# (oracle/_ref/muxsim, built by `make -C oracle`): trace.csv from
# gen-workload, records.csv from simulate with the hand-written plans.
set -euo pipefail
cd "$(dirname "$0")"
MUX=../../../oracle/_ref/muxsim
# b200prof: the pair config with the B200-measured LatencyProfile
# (profiles/r01_b200_profile_7b.json); its plan comes from the reference's own planner.
$MUX plan -c cfg_b200prof.json -o plan_b200prof.json > /dev/null
cp trace_pair.csv trace_b200prof.csv
for c in pair mesh b200prof empq; do
  [ $c = b200prof ] || $MUX gen-workload -c cfg_$c.json -o trace_$c.csv > /dev/null
  rm -rf out_$c
  $MUX simulate -c cfg_$c.json -p plan_$c.json -t trace_$c.csv -o out_$c > /dev/null
  mv out_$c/records.csv records_$c.csv
  mv out_$c/metrics.json metrics_$c.json
  mv out_$c/poolstats.json poolstats_$c.json
  rm -rf out_$c
done
