# certificates (fused mode) on the small configs: auto (off below 2^20 queries) vs on
set -x
for c in tiny depth lidar fragment; do
  for ce in 0 1; do
    echo "== $c cert=$ce"
    python bench.py --config $c --cert $ce --no-cpu-baseline --no-e2e --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read())
print(d['ms_per_step'], d['detail'].get('k3_total_ms'), d['detail'].get('fitness'), d['detail'].get('loop_ms'))"
  done
done
