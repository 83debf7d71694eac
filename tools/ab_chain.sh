for v in ${AB:-base pdl0t pdlp}; do
  TEMPO_B200_LIB=$PWD/_ab/$v/libtempo_b200.so timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'])"
done
