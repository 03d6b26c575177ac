#!/bin/bash
out=gpurun_out/r3b; mkdir -p $out
timeout 600 python scripts/e2e_host_profile.py > $out/e2e_host.json 2> $out/e2e_host.err; cat $out/e2e_host.json; tail -3 $out/e2e_host.err
MUX_GRAPHS=0 timeout 600 python scripts/e2e_host_profile.py > $out/e2e_host_nograph.json 2>&1; cat $out/e2e_host_nograph.json | tail -1
