import json, os, sys
d = json.loads(sys.stdin.read())
f = d["flagging"]
print(os.environ.get("V"), round(f["value"] / 1e9, 2), round(f["kernel_ms"], 4), round(f["full_span"]["value"] / 1e9, 2),
      round(f["full_span"]["kernel_ms"], 4), f["flagged"])
