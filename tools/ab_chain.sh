# Chain-level A/B: the bench.py chain (20 steps) per variant library built by
# tools/ab_build.sh NAME "-D...":   AB="base v1 v2" bash tools/ab_chain.sh
for v in ${AB:-base pdl0t pdlp}; do
  TEMPO_B200_LIB=$PWD/_ab/$v/libtempo_b200.so timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'])"
done
