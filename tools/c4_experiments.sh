#!/bin/bash
# Timing experiments on the threshold path (results invalid under PCWD_UNIT_DBG): where c4's time goes.
for dbg in 0 1 2 3; do
  PCWD_UNIT_DBG=$dbg python tools/launch_profile.py c4 f32 > gpurun_out/c4_dbg$dbg.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/c4_dbg$dbg.json')); print($dbg, round(d['step_ms'],2), [round(l['ms'],2) for l in d['launches']])"
done
for kb in 32 96 200; do
  PCWD_GENERIC_SMEM_KB=$kb python tools/launch_profile.py c4 f32 > gpurun_out/c4_smem$kb.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/c4_smem$kb.json')); print('smem $kb', round(d['step_ms'],2), [round(l['ms'],2) for l in d['launches']])"
done
