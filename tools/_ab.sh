timeout 800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c1 c2 c3 c4blk; do timeout 400 python tools/sweep.py --config $c --reps 40 --rounds 4 --variants '[{"variant":"xmarch"},{"variant":"xmarch","chunks":6},{"variant":"xmarch","chunks":4}]'; done
timeout 900 python tools/sweep.py --config c4full --step --reps 5 --rounds 2 --variants '[{"variant":"xmarch"},{"variant":"xmarch","chunks":1}]'
