# Copy one round measurement (scripts/gpu_round.sh output in gpurun_out/) into profiles/ under a round tag.
# usage: bash scripts/collect_profiles.sh r02
set -e
tag=${1:?round tag}
G=gpurun_out
P=profiles
for c in c0 c1 c2 c3 c4 ref_c1; do
  grep '^{' $G/bench_$c.log | tail -1 > $P/${tag}_bench_$c.json
done
cp $G/gpu_tests.log $P/${tag}_gpu_tests.log
cp $G/smoke.log $P/${tag}_smoke.log
cp $G/launches_c1.csv $P/${tag}_launches_c1.csv
cp $G/launches_c3.csv $P/${tag}_launches_c3.csv
for c in c0 c1 c3 c4; do cp $G/ncu_${c}_brief.txt $P/${tag}_ncu_$c.txt; done
for s in fd pd io td; do grep '^{' $G/side_$s.log | tail -1 > $P/${tag}_side_$s.json; done
grep '^{' $G/side_calls.log > $P/${tag}_side_calls.jsonl
ls -la $P/${tag}_*
