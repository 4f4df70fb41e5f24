#!/bin/bash
# Compact perf summary on one GPU: K1 in the c2 step (bench.py) and K4 (bench_step.py).
cd "$(dirname "$0")/.."
python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); r = d['roofline']
        print('c2 step: %.2f M rows/s  %.3f ms/step  K1 %.3f ms  %.0f GB/s  frac %.3f  clocks %s' % (
            d['value'] / 1e6, d['ms_per_step'], r['k1_ms'], r['achieved'], r['frac'], d['clocks']['sm_mhz']))"
python tools/bench_step.py 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l)
        print('K4 c3: cold %.1f us (%.0f GB/s, frac %.3f)  hot %.1f us' % (
            d['cold']['us_per_step'], d['cold']['gbs'], d['cold']['frac'], d['hot']['us_per_step']))"
