timeout 900 python -m pytest tests/test_channel_gpu.py tests/test_decode_gpu.py -q -m gpu --timeout 600 -p no:cacheprovider 2>&1 | tail -3
timeout 600 python tools/ber_bench.py > gpurun_out/ber_c5.json 2>gpurun_out/ber_c5.err; python -c "
import json; d=json.load(open('gpurun_out/ber_c5.json')); print({k:d[k] for k in ('seconds','frames_per_s','coded_Gbit_s')}); print(d['csv'])"; tail -3 gpurun_out/ber_c5.err
