import json, sys
for l in open(sys.argv[1]):
    if l.startswith('{"kind"'):
        d = json.loads(l); e = d["env"]
        print(e.get("SEQCDC_LIB", "")[6:], e.get("SEQCDC_WALKERS_PER_SM", ""), d["kind"], d["MiB"], d["GBps"], d["walk_GBps"])
    elif l.startswith('{"MiB"'):
        d = json.loads(l); print("  lone seg", d["seg_MiB"], "us/chunk", d["us_per_chunk_per_walker"], "GBps", d["GBps"])
    else:
        print(l.rstrip())
