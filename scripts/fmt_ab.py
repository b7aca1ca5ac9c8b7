import sys, json
for ln in sys.stdin:
    if ln.startswith('{'):
        d = json.loads(ln)
        print(d['n'], d['precision'], 'persistent %.4f (%.2f)' % (d['persistent']['device_ms'], d['persistent']['roofline_frac']), 'tiled %.4f (%.2f)' % (d['tiled']['device_ms'], d['tiled']['roofline_frac']), 'wall', round(d['persistent']['wall_ms'],3), round(d['tiled']['wall_ms'],3), d['persistent']['launches'])
    else:
        print(ln.rstrip()[:300])
