#!/usr/bin/env bash
# The reference's own simulator (baseline/_ref, unmodified prefillsim CLI) on its post-rec trace, one instance,
# H100 preset: P99 and mean latency of FIFO, SRJF and calibrated SRJF at rates around saturation. Shows that the
# policy ordering at P99 (FIFO >= SRJF past the knee) is the reference's, not an artefact of this build.
cd "$(dirname "$0")/.."
for pol in fifo srjf srjf-calibrated; do
  PYTHONPATH=baseline/_ref python -c "import sys; from prefillsim.cli import main; sys.exit(main(sys.argv[1:]))" \
    simulate --gpu h100 --policy $pol --multipliers 0.5,0.8,0.9,1,1.1,1.2,1.5,2 --instances 1 | \
    { [ "$pol" = fifo ] && cat || tail -n +2; }
done
