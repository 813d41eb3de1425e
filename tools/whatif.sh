# What-if timing: the bench step with each kernel category dropped (DPB_SKIP_MASK; results invalid).
for m in 0 4 8 16 32 128 1024 832 512 64 256; do
  v=$(DPB_SKIP_MASK=$m timeout 300 python bench.py --no-cpu-baseline --no-naive --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3))")
  echo "mask $m ms_per_step $v"
done
