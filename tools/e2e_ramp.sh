#!/bin/bash
# e2e time of SweepSolver.sweep (pageable numpy, reused output) for several block ramps (HSW_E2E_RAMP)
for r in "$@"; do
  echo "== ramp $r"
  HSW_E2E_RAMP=$r timeout 300 python tools/e2e_probe.py c4 2>&1 | grep "reused-output" | tail -1
done
