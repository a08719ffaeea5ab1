"""A stand-in serving program for dispatcher tests (no GPU): prints READY,
answers grpc-style health/info frames and REST /health, records its
CUDA_VISIBLE_DEVICES into --record."""
import argparse
import json
import os
import socketserver
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2006_05096_b200 import wire  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model")
ap.add_argument("--protocol")
ap.add_argument("--record")
args = ap.parse_args()
Path(args.record).write_text(os.environ.get("CUDA_VISIBLE_DEVICES", "<unset>"))


class H(socketserver.BaseRequestHandler):
    def handle(self):
        while True:
            raw = wire.read_frame(self.request)
            if raw is None:
                return
            msg = json.loads(raw)
            wire.write_frame(self.request, json.dumps({"ok": True, "kind": msg.get("kind")}).encode())


class S(socketserver.ThreadingTCPServer):
    daemon_threads = True
    allow_reuse_address = True


srv = S(("127.0.0.1", 0), H)
print(f"READY {srv.server_address[1]}", flush=True)
srv.serve_forever()
