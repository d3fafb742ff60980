# config table (per-call synced with graphs warmed + back-to-back graph / direct)
set -x
timeout 1200 python scripts/config_table.py > gpurun_out/configs_r2k.md 2> gpurun_out/configs_r2k.err; cat gpurun_out/configs_r2k.md
tail -3 gpurun_out/configs_r2k.err
