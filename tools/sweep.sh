#!/bin/bash
# usage: tools/sweep.sh "<cfgs>" "opts1" "opts2" ...   (each opts: "name=value name=value")
cfgs="$1"; shift
for o in "$@"; do
  args=""
  for kv in $o; do args="$args --opt $kv"; done
  echo "### $o"
  python tools/run_workload.py $cfgs --repeat ${REPEAT:-1} $args 2>&1 | python -c "
import sys, json
for line in sys.stdin:
    try: r = json.loads(line)
    except Exception: print(line.strip()); continue
    if r.get('rep', 0) != int('${REPEAT:-1}') - 1: continue
    s = r['stats']
    print('cfg%d pos=%s ok=%s prep=%.1fms search=%.1fms scan=%.1fms calls=%.3g terms=%.3g batches=%d scanned=%d launches=%d terms/s=%.3g live/tile=%.1f chunks/tile=%.2f lb_skipped=%.3g dot=%d/%d' % (r['cfg'], r['positions'][:2], r['golden_match'], s['prep_ms'], s['search_ms'], s['scan_kernel_ms'], s['calls'], s['terms'], s['batches'], s['scanned_candidates'], s['kernel_launches'], r['terms_per_s'], s['tile_live_candidates']/max(1,s['tiles']), s['scan_kernel_terms']/max(1,s['tiles'])/(128*64*64), s['lb_skipped'], s.get('scan_kernel_dot_launches',0), s['scan_kernel_launches']))
"
done
