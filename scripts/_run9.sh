set -u
O=gpurun_out/r2m
mkdir -p $O
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"
bash scripts/profile_round.sh $O/prof; echo "prof rc=$?"
