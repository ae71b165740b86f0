timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_tests.log
V='[{"variant":"xmarch"},{"variant":"xmarch_generic"},{"variant":"xmarch"},{"variant":"xmarch_generic"}]'
for c in c1 c2 c3 c4blk; do
 for L in paper_2010_01545_b200/libpwadv.so build/variants/libpwadv_sleep2k.so build/variants/libpwadv_sleep200.so; do
  PWADV_LIB=$L timeout 300 python tools/sweep.py --config $c --reps 200 --variants "$V" | python -c "
import sys,json
for d in map(json.loads, sys.stdin):
    print('$c', '$L'.split('/')[-1], d['variant'] if isinstance(d['variant'],str) else d['variant'].get('variant'), d.get('gpts'), d.get('bitwise_same_as_first'))"
 done
done
