"""The reference-side binding (integration/oscfield_gpu_seams.cpp) compiles against the
reference's own headers and links against the C-ABI, and the resulting program runs the
reference's types through the seam. CPU test: compiles and links only (no GPU call)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_seams_compile_against_reference_headers(tmp_path, P):
    obj = tmp_path / "seams.o"
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-fPIC", "-Wall", "-Wextra", "-Werror", "-I", REF_INC,
                    "-I", os.path.join(ROOT, "include"), "-c",
                    os.path.join(ROOT, "integration", "oscfield_gpu_seams.cpp"), "-o", str(obj)],
                   check=True)
    # link into a shared object against libosc_b200.so: every C-ABI symbol used must resolve
    so = tmp_path / "libseams.so"
    subprocess.run(["/usr/bin/g++", "-shared", "-o", str(so), str(obj),
                    "-L", os.path.join(ROOT, "paper_2306_13493_b200"), "-losc_b200",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_2306_13493_b200")],
                   check=True)
    nm = subprocess.run(["nm", "-DC", str(so)], capture_output=True, text=True).stdout
    assert "oscfield::run_level_draws" in nm and "oscfield::summarize_draws" in nm
