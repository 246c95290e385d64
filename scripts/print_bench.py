import sys, json
tag = sys.argv[1]
r = json.loads(sys.stdin.read())
print("graphs", tag, "value", round(r["value"], 4), "setup", round(r["setup_s"], 4), "solve", round(r["solve_s"], 4), "its", r["its"], "launches", r["gpu_launches"], "e2e", round(r["e2e"]["value"], 4))
