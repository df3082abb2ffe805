# Per-CTA timelines (trace build) of cfg2 and cfg1 T=8/T=32 steps.
set -x
O=gpurun_out/r2m
mkdir -p $O
timeout 300 python tools/trace_timeline.py --scenario cfg2,t8,t8flush,t32 --reps 2 > $O/timeline.log 2>&1
ls -la $O
