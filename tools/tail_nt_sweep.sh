#!/bin/bash
# Timing experiment: threads per unit of the coarse tail kernel (PCWD_TAIL_NT), c5 decompose median (no L2 flush)
for nt in 256 128 64 256 128 64; do
  echo -n "$nt "; PCWD_TAIL_NT=$nt python tools/skip_timing.py c5
done
