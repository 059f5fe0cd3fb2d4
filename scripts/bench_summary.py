"""Print the headline numbers of bench.py JSON lines (one file per argument)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unparseable:", e)
        continue
    r = d.get("roofline") or {}
    print(f"{path}: {d.get('workload')} value {d['value']:.1f} e2e {d['e2e']['value']}"
          f" ms/pair {d.get('ms_per_pair')} top {r.get('group')} frac {r.get('frac')}")
    print("  stages:", {k: round(v['us_per_pair'], 1) for k, v in r.get('stages', {}).items()})
    print("  groups:", {k: (round(v['avg_launch_ms'], 3), round(v['frac'], 3),
                            round(v['share_of_chain'] or 0, 3))
                        for k, v in r.get('kernel_groups', {}).items()})
    print("  pipe roofline:", {k: (v['pipe_roofline']['binding_pipe'],
                                   round(v['pipe_roofline']['frac'], 3))
                               for k, v in r.get('kernel_groups', {}).items() if 'pipe_roofline' in v})
    print("  parity:", d.get("parity"), "clocks:", d.get("clocks"))
    if d.get("cpu_baseline"):
        print("  cpu:", {k: d['cpu_baseline'].get(k) for k in ('value', 'cores', 'kind')})
