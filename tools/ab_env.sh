#!/bin/bash
# A/B over environment knobs: each line of stdin "NAME VAR=VAL ..." runs ab_pulse
# on CONFIG for the dense prefix (20 pulses from 5) and the full arc.
cfg=${1:-3}; full=${2:-256}
while read -r name envs; do
  a=$(env $envs START=5 python tools/ab_pulse.py $cfg 20 q | grep pulses/s)
  b=$(env $envs python tools/ab_pulse.py $cfg $full | tr '\n' ' ')
  echo "$name | $envs | dense20: $a | full: $b"
done
