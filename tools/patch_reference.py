#!/usr/bin/env python3
"""Applies INTEGRATION.md's patch to a COPY of the reference tree: one more engine, `cuda`,
behind tsdd::run_discovery, bound to libtsdd_cuda.so through include/tsdd/cuda_engine.hpp.

    python tools/patch_reference.py /root/reference/proj /tmp/proj_cuda

The reference itself is never written to.  Four edits, each anchored on a line of the
reference and checked to apply exactly once:
  1. include/tsdd/discovery.hpp:16   enum class Engine gains `cuda`
  2. src/discovery.cpp:102-112       engine_name() names it
  3. src/pipeline.cpp:12-17          parse_engine() accepts "cuda"
  4. src/pipeline.cpp:53-54          run_discovery() hands Engine::cuda to tsdd::cuda::run_discovery
     before the CPU preparation stage (the CUDA engine prepares on the device), and the engine
     switch (:78-88) gets an empty case for it
"""
import os
import shutil
import sys


def edit(path: str, old: str, new: str) -> None:
    text = open(path).read()
    if text.count(old) != 1:
        raise SystemExit(f"{path}: expected exactly one occurrence of {old!r}, found {text.count(old)}")
    with open(path, "w") as f:
        f.write(text.replace(old, new))


def main() -> None:
    if len(sys.argv) != 3:
        raise SystemExit(__doc__)
    src, dst = sys.argv[1], sys.argv[2]
    if os.path.exists(dst):
        shutil.rmtree(dst)
    shutil.copytree(src, dst)
    for root, _, files in os.walk(dst):  # the reference tree is read-only; its copy must not be
        os.chmod(root, 0o755)
        for name in files:
            os.chmod(os.path.join(root, name), 0o644)

    edit(os.path.join(dst, "include/tsdd/discovery.hpp"),
         "enum class Engine { brute, hotsax, phidd };",
         "enum class Engine { brute, hotsax, phidd, cuda };")
    edit(os.path.join(dst, "src/discovery.cpp"),
         '      return "phidd";\n',
         '      return "phidd";\n    case Engine::cuda:\n      return "cuda";\n')
    pipeline = os.path.join(dst, "src/pipeline.cpp")
    edit(pipeline,
         '#include "tsdd/pipeline.hpp"\n',
         '#include "tsdd/pipeline.hpp"\n\n'
         '#define TSDD_CUDA_WITH_REFERENCE_HEADERS  // cuda_engine.hpp then uses this tree\'s own types\n'
         '#include "tsdd/cuda_engine.hpp"           // from the B200 engine\'s include/\n')
    edit(pipeline,
         '  if (name == "phidd") return Engine::phidd;\n',
         '  if (name == "phidd") return Engine::phidd;\n  if (name == "cuda") return Engine::cuda;\n')
    edit(pipeline,
         "RunOutcome run_discovery(const TimeSeries& series, const DiscoveryConfig& config) {\n",
         "RunOutcome run_discovery(const TimeSeries& series, const DiscoveryConfig& config) {\n"
         "  // validates like check_config (same order and messages; dictionary guard 2^32), prepares and\n"
         "  // searches on the device, throws this tree's exception types\n"
         "  if (config.engine == Engine::cuda) return tsdd::cuda::run_discovery(series, config);\n")
    edit(pipeline,
         "      outcome.result = phidd_discord(matrix, indexes, options);\n      break;\n",
         "      outcome.result = phidd_discord(matrix, indexes, options);\n      break;\n"
         "    case Engine::cuda:\n      break;  // returned above\n")
    print(dst)


if __name__ == "__main__":
    main()
