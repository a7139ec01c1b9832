import json, sys
for f in sys.argv[1:]:
    for l in open(f):
        d = json.loads(l)
        print('==', d['case'], d['dtype'], d['env'])
        for r in d['rows']:
            if 'us' in r: print(f"  L{r['level']} k{r['kind']} nv{r['nv']}: {r['us']:8.2f} us {r['GBps']:8.1f} GB/s")
            elif 'vcycle_ms' in r: print(f"  L{r['level']} vcycle {r['vcycle_ms']} ms")
