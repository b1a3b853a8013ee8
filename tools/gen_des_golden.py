"""Generates tests/golden/des_sha256.json: sha256 + record count of the reference simulator's
event log (oracle/_ref/ref_des, the unmodified reference pool) for every scenario x preset.
Run in the container that has /root/reference (after `make -C oracle`)."""
import hashlib
import json
import os
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import des_cases  # noqa: E402

out = {}
with tempfile.TemporaryDirectory() as td:
    for scen, preset in des_cases.cases():
        path = os.path.join(td, "e.jsonl")
        r = subprocess.run([os.path.join(des_cases.REF_DIR, "ref_des"),
                            os.path.join(des_cases.SCEN, scen + ".json"), path, preset],
                           capture_output=True, text=True, check=True)
        data = open(path, "rb").read()
        out[f"{scen}/{preset}"] = {"sha256": hashlib.sha256(data).hexdigest(),
                                   "bytes": len(data), "records": data.count(b"\n")}
        print(scen, preset, out[f"{scen}/{preset}"]["records"], flush=True)
json.dump(out, open(os.path.join(des_cases.ROOT, "tests", "golden", "des_sha256.json"), "w"), indent=1,
          sort_keys=True)
