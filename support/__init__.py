"""Test and benchmark support (input generators).  Not part of the product
package: nothing under paper_2210_14771_b200/ imports it."""
