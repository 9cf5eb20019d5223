"""Print the search.* / build phase times of tools/run_case.py JSON outputs."""
import json
import sys

for f in sys.argv[1:]:
    s = open(f).read()
    try:
        d = json.loads(s[s.index("{"):])
    except ValueError:
        print(f, "unparsable:", s[-300:])
        continue
    ph = d.get("phases_ms", {})
    keep = {k: round(v, 3) for k, v in ph.items() if k.startswith("search") or k.startswith("density")}
    keep["build"] = round(sum(v for k, v in ph.items() if k.startswith("build.")), 3)
    print(f.split("/")[-1].ljust(18), keep)
