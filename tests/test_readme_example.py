"""The README's API example runs as written (GPU)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_readme_python_example_runs(capsys):
    text = open(os.path.join(ROOT, "README.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    assert blocks, "README has no python example"
    exec(compile(blocks[0], "README.md", "exec"), {})
    out = capsys.readouterr().out
    assert "[" in out                      # the printed commit order
