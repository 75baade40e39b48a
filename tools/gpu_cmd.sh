timeout 600 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -x 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(check|var|node)" -c 40 --csv --log-file gpurun_out/launches_x.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
bash profiles/variants.sh
