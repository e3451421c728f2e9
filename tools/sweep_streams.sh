# bench throughput over (streams, views per step): bash tools/sweep_streams.sh "8 12 16" "16 32"
for s in ${1:-4 8}; do for v in ${2:-8 16}; do
python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e --no-others --streams $s --views $v 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('streams $s views $v', round(d['value']))"
done; done
