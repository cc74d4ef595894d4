"""Print one key of a bench JSON line: python tools/show.py FILE KEY"""
import json
import sys

print(json.dumps(json.load(open(sys.argv[1])).get(sys.argv[2])))
