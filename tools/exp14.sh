for rep in 1 2; do
echo "c3 dense $(timeout 300 python tools/prof_round.py --config c3 --reps 3 --debug-flags 0x1000 --solve 2>&1 | tail -1)"
echo "c3 worklist $(timeout 300 python tools/prof_round.py --config c3 --reps 3 --debug-flags 0x1000 --solve --worklist 2>&1 | tail -1)"
done
