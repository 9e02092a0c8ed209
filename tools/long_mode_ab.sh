#!/bin/sh
# A/B of the long-row paths on cfg4-style matrices (tools/cfg4_split.py)
for cfg in "0 4 64" "1 4 64" "2 4 64" "2 4 64" "2 4 128" "1 4 128"; do
  set -- $cfg
  echo "== SELLB_LONG_MODE=$1 LONG_D=$2 GRP_SB=$3"
  SELLB_LONG_MODE=$1 SELLB_LONG_D=$2 SELLB_GRP_SB=$3 timeout 120 python tools/cfg4_split.py
done
