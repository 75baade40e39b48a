python tools/membench.py > gpurun_out/membench.json 2>&1; cat gpurun_out/membench.json
LDPC_SLOTS=var timeout 600 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -x 2>&1 | tail -2
EXTRA_VARIANTS="LDPC_SLOTS=var LDPC_KERNEL=pipe,LDPC_SLOTS=var" bash profiles/variants.sh
