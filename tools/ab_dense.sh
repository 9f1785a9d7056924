#!/bin/bash
# dense-window-only A/B (pulses 5..24 of CONFIG): stdin lines "NAME VAR=VAL ..."
cfg=${1:-3}
while read -r name envs; do
  a=$(env $envs START=5 python tools/ab_pulse.py $cfg 20 q | grep pulses/s)
  echo "$name | $envs | dense20: $a"
done
