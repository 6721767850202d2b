"""Golden digest of the reference's N2FW checkpoint (model.save_checkpoint,
model.py:143-152) of the seeded networks ``build_network(1, seed)``:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_checkpoint.py

Writes ``tests/golden/checkpoint_digests.json`` (SHA-256 and size of the
file bytes; the files themselves are 4.7 MB each and stay out of the repo).
"""

import hashlib
import json
import os
import sys
import tempfile

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "checkpoint_digests.json")


def main():
    sys.path.insert(0, REF)
    from noise2fast import model  # noqa: E402

    out = {}
    for seed in (0, 7, 4242):
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "w.n2fw")
            model.save_checkpoint(model.build_network(1, seed), path)
            data = open(path, "rb").read()
        out[str(seed)] = {"sha256": hashlib.sha256(data).hexdigest(), "bytes": len(data),
                          "header_hex": data[:28 + 16 * 9 + 8].hex()}
    json.dump(out, open(OUT, "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main()
