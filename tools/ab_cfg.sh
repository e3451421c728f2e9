# A/B library builds on one config: bash tools/ab_cfg.sh "<bench args>" lib1.so lib2.so ...
args=$1; shift
for lib in "$@"; do
  GES_B200_LIB=$lib python bench.py $args --steps 20 --warmup 3 --no-cpu --no-e2e --no-others 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$lib', '$args', round(d['value']))"
done
