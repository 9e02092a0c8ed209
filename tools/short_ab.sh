#!/bin/sh
for env in "SELLB_SHORT=0" "SELLB_SHORT_K=2" "SELLB_SHORT_K=4" "SELLB_SHORT_K=8"; do
  echo "== $env"; env $env python tools/short_probe.py
done
