# one bench line reduced to "config value ms": bash tools/bval.sh C2 [steps]
timeout 600 python bench.py --config $1 --steps ${2:-5} --warmup 3 --no-cpu-baseline 2>/dev/null | \
python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value'],3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
