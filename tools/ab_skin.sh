B=128 SKINS=0.25,0.15,0.2,0.25,0.35 timeout 900 python tools/prof_skin.py 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(d['skin'], d['reg_per_s'], d['s'], 'sweep_ms', d['sweep_ms'], 'builds', {k:v for k,v in d.get('builds',{}).items() if k in ('build_ms','grid_builds','filter_builds')})
"
