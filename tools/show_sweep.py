import json, sys
for line in open(sys.argv[1]):
    if line.startswith('=='): print(line.strip()); continue
    try: d = json.loads(line)
    except Exception: print(line.strip()[:200]); continue
    for p in ('hot', 'random'):
        if p not in d: continue
        r = d[p]; t = r.get('trace_us', {})
        print(f"   {p:6s} graph_us {r['graph_us']:.2f} GBps {r['graph_GBps']:.0f} "
              + " ".join(f"{k}={v}" for k, v in t.items() if k in ('first_page', 'consumed', 'pdl_passed', 'merged', 'inbox', 'exit', 'sm_mhz', 'cycles_spin_write_merge_push_arrive')))
