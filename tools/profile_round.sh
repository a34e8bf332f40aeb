# Round profile set: bench line, launch list of one live frame, ncu --set full
# of the frame's fallback traversal launches (the dominant stage).
# Usage: bash tools/profile_round.sh <tag>
set -e
tag=${1:-r1}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
python bench.py --profile-only --warmup 1 > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --profile-only --warmup 1 > /dev/null 2>&1
# workload generation traces twice (primary, bounce hit frames); the frame's
# three fallback-queue traversals follow
ncu --set full --import-source on --clock-control none -k regex:k_trace -s 2 -c 3 \
    -o gpurun_out/trace_$tag python bench.py --profile-only --warmup 1 > /dev/null 2>&1
tail -c 400 gpurun_out/bench_$tag.json
