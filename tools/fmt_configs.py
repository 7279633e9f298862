import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    for k,v in d.items():
        if isinstance(v,dict) and "gpu" in v: print(d["config"], k, round(v["gpu"]["ids_per_s"]/1e6,1), "M/s", round(v["gpu"]["ms_per_batch"],3), v["gpu"]["outcomes"], "ref", round(v["reference"]["ids_per_s"]/1e6,1))
