for s in 0 16 32 48 64; do echo "dbg $s"; PCWD_UNIT_DBG=$s python tools/launch_profile.py c4 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print([ (l['level'], l['ms']) for l in d['launches']])"; done
