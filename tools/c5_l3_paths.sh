# c5 level-3 path experiments: fine (wide / narrow), tile, batched
run() { echo "$1"; env $1 python tools/launch_profile.py c5 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['step_ms'],3), round(d['step_ms_serialised'],3), [ (l['kind'], l['level'], l['ms']) for l in d['launches'] if l['level'] <= 4])"; }
run "X=0"
run "PCWD_FINE_WIDE=0"
run "PCWD_FINE_WIDE=7"
run "PCWD_FINE_MAXLEV=2"
run "PCWD_FINE_MAXLEV=2 PCWD_NO_TILE=1"
