"""TEST INFRASTRUCTURE ONLY — the REAL reference behind pyoracle's interface.

``oracle/_ref/libntf_ref.so`` is the reference's own unmodified sources
(/root/reference/proj/src/*.cpp) compiled by ``oracle/ref_build/Makefile``
against a small Eigen stand-in (Eigen3 is not in this image); its C surface
(``oracle/ref_build/ref_capi.cpp``) exports the same symbols as the oracle's.
This module is a second instance of ``pyoracle`` bound to that library, so

    import pyoracle as O, pyref as R
    O.run("her", t, init, ...)   # the restatement
    R.run("her", t, init, ...)   # the reference itself

take identical arguments. Only tests/ and bench.py's CPU legs import it.
``available()`` is False when the library has not been built and
/root/reference is absent (nothing can build it then).
"""
import importlib.util as _ilu
import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))
REF_ROOT = "/root/reference/proj"
LIB_PATH = _os.path.join(_HERE, "_ref", "libntf_ref.so")


def available():
    return _os.path.exists(LIB_PATH) or _os.path.isdir(REF_ROOT)


_spec = _ilu.spec_from_file_location("_pyref_impl", _os.path.join(_HERE, "pyoracle.py"))
_impl = _ilu.module_from_spec(_spec)
_spec.loader.exec_module(_impl)
_impl._LIB_FILE = _os.path.join("_ref", "libntf_ref.so")

for _name in dir(_impl):
    if not _name.startswith("_"):
        globals()[_name] = getattr(_impl, _name)


def is_reference_build():
    return bool(_impl.lib().ora_is_reference_build())
