# A/B of the stacked-launch schedule's cost-model constants (development probe)
for wl in config4 config3 config5; do
  for f in 0 4 0 4; do
    FLASHHE_REL_FILL_US=$f timeout 300 python bench.py --workload $wl --no-e2e --no-sub --no-cpu --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fill $f', d['config']['workload'][:8], d['ms_per_step'], d['roofline']['frac'])"
  done
done
