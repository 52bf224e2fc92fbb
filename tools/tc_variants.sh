for v in inl64 iss64 iss128 inl128; do echo "== $v"; QB_LIB_PATH=build/exp/libqb_$v.so timeout 200 python tools/tc_check.py E:38 E:40 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['n'], d['ok'], 'coarse', round(d['coarse_ms'],2), 'tc', round(d['tc_ms'],2), 'grid', d['grid'], 'k', d['k_tc'])
    else: print(l.strip())
"; done
