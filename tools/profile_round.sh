# Round profile set on the headline config (BASELINE c5 by default):
#   * the launch list of one live frame (ncu gpu__time_duration.sum,
#     cold-cache and serialised: shares, not absolute times),
#   * ncu --set full of the frame's fallback traversals (the dominant stage),
#     the hash kernel and the largest consult kernels,
#   * per-launch DRAM traffic of the traversal (profiles/traffic.json).
# Each ncu command runs only after the same program exited 0 without ncu.
# Usage (on the GPU box): bash tools/profile_round.sh <tag> [config]
set -e
tag=${1:-r2}
cfg=${2:-c5}
out=gpurun_out/prof_$tag
mkdir -p $out
python tools/frame_profile.py $cfg live 1 > $out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $out/launches_$cfg.csv python tools/frame_profile.py $cfg live 1 > /dev/null 2>&1
# the workload's spawning traversals come first (one per bounce level)
skip=$(python -c "from paper_1910_01304_b200.scenes import make_scene; print(make_scene('$cfg', resolution=(8, 8)).bounces + 1)")
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:"k_trace" --launch-skip $skip --csv \
    --log-file $out/trace_traffic_$cfg.csv python tools/frame_profile.py $cfg live 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_trace" --launch-skip $skip \
    -c 3 -o $out/trace_$cfg python tools/frame_profile.py $cfg live 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none \
    -k regex:"k_hash_bulk|k_eval0|k_finalize|k_replay_block|k_commit_apply|k_seg_lookup|k_first_append" \
    -c 12 -o $out/consult_$cfg python tools/frame_profile.py $cfg live 1 > /dev/null 2>&1
echo done
