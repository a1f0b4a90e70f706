#!/usr/bin/env python3
"""The reference's own command line (`linevox render|serve ...`, lv/cli.py) on the B200 pipeline: imports the
unmodified reference package from baseline/_ref, points its `ScenePipeline` at paper_2510_09081_b200.ScenePipeline
and hands over to its `main()`.  Everything else -- argument parsing, config files, PPM/HITI/stats/dump writing,
the websocket protocol -- is the reference's code.

    python tools/reference_frontend.py render --input gen:random_streamlines?polylines=100&verts_per_line=101 \\
           --res 64 --strategy vcsv --width 256 --height 256 --out /tmp/frame --dump
    python tools/reference_frontend.py serve --input scene.lns --res 256 --width 1920 --height 1080 --port 8765
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))


def main(argv=None) -> int:
    try:
        import linevox.cli
        import linevox.pipeline
        import linevox.server
    except ImportError as e:
        print(f"the reference package is not installed under baseline/_ref ({e}); run __graft_entry__.build() "
              "where /root/reference exists", file=sys.stderr)
        return 2
    import paper_2510_09081_b200 as lvx
    linevox.pipeline.ScenePipeline = lvx.ScenePipeline      # lv/cli.py:67 imports the name at call time
    linevox.server.ScenePipeline = lvx.ScenePipeline        # lv/server.py:21 holds its own reference
    return linevox.cli.main(argv)


if __name__ == "__main__":
    sys.exit(main())
