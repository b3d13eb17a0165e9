python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 8 16 24 16; do
  DISC_S2_SMS=$r python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('res $r', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['avg_launch_ms'],3), round(d['path_roofline']['stage1_ms']/10,3), round(d['path_roofline']['stage2_ms']/10,3), d['m1']['value'])"
done
