set -u
O=gpurun_out/r2b
mkdir -p $O
bash scripts/fullsize_round.sh $O/fs
bash scripts/sanitize_round.sh $O/san
