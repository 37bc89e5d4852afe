for cfg in "RS_FAST_STEP=0" "RS_FC_HMINB=5" "RS_FC_HMINB=2" "RS_FC_HMINB=5"; do
  echo "$cfg $(env $cfg timeout 300 python tools/exp_flush.py 30 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print([round(x["median_ms"]*1e3,1) for x in d["dirty"]+d["clean"]])')"
done
