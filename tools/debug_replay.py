"""Debug helper: run a few golden cases through the device replay one at a time."""
import sys, json
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from golden_cases import cases, config_from, trace_from
from paper_2602_03921_b200 import _device
from paper_2602_03921_b200.records import canon_reference_record, digest_records
names = sys.argv[1:] or [c["name"] for c in cases()[:40]]
for name in names:
    c = next(x for x in cases() if x["name"] == name)
    b = _device.ReplayBatch([config_from(c)], [trace_from(c["trace"])], full_log=True)
    b.launch()
    r = b.results()[0]
    canon = [canon_reference_record(x) for x in r.log]
    ok = json.dumps(r.report) == json.dumps(c["report"]) and digest_records(canon) == c["log_sha256"]
    print(name, "OK" if ok else "MISMATCH", len(canon), c["log_len"], flush=True)
    if not ok and "log" in c:
        for i, (a, g) in enumerate(zip(canon, c["log"])):
            if list(a) != g:
                print("  first diff", i, a, g); break
