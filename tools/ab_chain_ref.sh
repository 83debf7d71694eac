# chain with the reference's mask stream generated every step, per variant
for v in ${AB:-base}; do
  TEMPO_B200_LIB=$PWD/_ab/$v/libtempo_b200.so timeout 300 python bench.py --masks reference --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], d['reference_mask_generation']['ms'])"
done
