# hybrid generic-kernel scratch (steps >= 2 in shared memory) vs all-global, c4 launch profiles
for kb in 40 64 0; do echo "hybrid cap $kb KB"; PCWD_HYBRID_KB=$kb python tools/launch_profile.py c4 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['step_ms'], d['step_ms_serialised'], [ (l['level'], l['ms']) for l in d['launches']])"; done
