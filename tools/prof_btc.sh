python tools/bt_dbg.py 2>&1 | tail -3
python tools/batched_engines.py
for p in 1 2 3; do echo "per_sm=$p"; CPA_SVT_BTC_PER_SM=$p python tools/batched_engines.py | tail -1; done
