for c in 2 5 6; do
python tools/phase_times.py --config $c --reps 5 2>/dev/null | tail -1
python tools/phase_times.py --config $c --reps 5 --reuse-poly 2>/dev/null | tail -1
done
