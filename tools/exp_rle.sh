#!/bin/bash
for dbg in 0 1; do
  echo "=== CDM_DEBUG_RLE=$dbg"
  CDM_SERIAL=1 CDM_DEBUG_RLE=$dbg timeout 300 python tools/trace_rle.py 2>&1 | grep -A3 "('rle'"
done
