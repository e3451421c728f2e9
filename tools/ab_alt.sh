# A/B builds of the library, alternating: bash tools/ab_alt.sh lib1.so lib2.so ... (3 rounds)
for i in 1 2 3; do for lib in "$@"; do
GES_B200_LIB=$lib python bench.py --steps 60 --warmup 3 --no-cpu --no-e2e --no-others 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$lib', round(d['value']), round(d['roofline']['frame_ms']*1000,1), {k:round(v*1000,1) for k,v in d['roofline']['phase_ms'].items()})"
done; done
