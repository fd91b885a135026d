# closing pass: every -m gpu test, smoke, the default bench line, then the sanitizers over every kernel family
bash tools/gpu_full.sh
bash tools/gpu_sanitize.sh
