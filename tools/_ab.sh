timeout 800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c1 c2 c3 c4blk; do timeout 400 python tools/sweep.py --config $c --reps 50 --rounds 3 --variants '[{"variant":"xmarch"}]'; done
python bench.py --steps 1000 --no-e2e --no-cpu | cut -c1-200
