# RSim row kernel: TMA-staged (default) vs register fallback (CEL_RSIM=0), one B200
for v in 5 0; do
  r=$(CEL_RSIM=$v timeout 120 python bench_config.py --workload rsim --gpus 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.0f rows/s rsim_row %.1f ms' % (d['value'], d['profile_ms']['rsim_row']['ms']))")
  echo "variant=$v $r"
done
