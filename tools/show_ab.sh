for f in "$@"; do grep -v Warn $f | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    km=d.get('kernels_ms') or {}
    print(' '.join(f'{k}={d[k]}' for k in d if k in ('l1','l2','ms','total_ms')), ' | ', ' '.join(f'{k.split(\"(\")[0].replace(\"void sg::\",\"\")}={v}' for k,v in km.items()))
"; done
