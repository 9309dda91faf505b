#!/bin/sh
# Install the UNMODIFIED reference (serve_emu) into baseline/_ref (git-ignored; it
# travels to the GPU box with gpurun).  Built from a /tmp copy because setuptools
# writes into the source tree; --no-deps because its dependencies (numpy, fastapi,
# uvicorn, httpx) are already in this image and pip cannot resolve them offline.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
rm -rf /tmp/serve_emu_build "$HERE/_ref"
cp -r /root/reference/pkg /tmp/serve_emu_build
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$HERE/_ref" /tmp/serve_emu_build
