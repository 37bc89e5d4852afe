for cfg in "RS_FAST_STEP=0" "RS_FAST_PRIO=hh" "RS_FAST_PRIO=nn" "RS_FAST_PRIO=nh" "RS_FAST_PRIO=hn" "RS_FAST_PRIO=nh RS_FCH_ITEMS=1184" "RS_FAST_PRIO=nh RS_FCH_ITEMS=4736" "RS_FAST_PRIO=hh"; do
  echo "$cfg $(env $cfg timeout 300 python tools/exp_flush.py 30 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print([round(x["median_ms"]*1e3,1) for x in d["dirty"]+d["clean"]])')"
done
