for r in 1 2 3; do
for L in old b200; do
MCF_LIB=$PWD/paper_2207_08867_b200/libmcf_$L.so python bench.py --steps 20 --warmup 5 --no-extras 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']
print('$L', d['ms_per_step'], {a:b['ms'] for a,b in k.items()})"
done; done
