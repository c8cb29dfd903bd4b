"""Legacy VTK writer under the reference's module name
(/root/reference/pkg/src/fedheat/vtkio.py:20-57); the implementation is in
`output.py` (native number formatting)."""

from .output import vtk_text, write_vtk

__all__ = ["vtk_text", "write_vtk"]
