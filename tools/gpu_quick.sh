set -o pipefail
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --no-cpu-baseline --no-extra > gpurun_out/bq.json 2> gpurun_out/bq.err; echo bench rc=$?
