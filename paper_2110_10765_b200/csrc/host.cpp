// Host half of the C-ABI: error state, work-unit planning and GPU partitioning.
//
// cim_plan_units is the native replacement for the reference's per-(tile,row)
// segment bookkeeping (CountsAndOffsets, scan.py:45-65, built through
// counts_to_offsets at pipeline.py:319-330): instead of one segment per state
// row, the B200 layout needs one work unit per run of ≤ max_unit tiles of a
// block row, which is what the persistent kernel schedules.
#include <cstdint>
#include <string>
#include <vector>

#include "cim_b200.h"
#include "host_util.h"

namespace cim {
namespace {
thread_local std::string g_last_error;
}
int set_error(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}
void clear_error() { g_last_error.clear(); }
}  // namespace cim

using cim::set_error;

extern "C" const char *cim_version(void) { return "cim_b200 1.0 (sm_100a, fragment layout v1)"; }

extern "C" const char *cim_last_error(void) { return cim::g_last_error.c_str(); }

// Tiles must be grouped by column band (band = C / band_cols, ascending), and
// inside a band sorted by R then C, unique, R ≤ C.  band_cols ≥ nb is the
// plain row-major order.  Units never cross a band or a block row.
extern "C" int cim_plan_units_banded(const int32_t *rc, int64_t n_tiles, int64_t nb, int32_t max_unit,
                                     int64_t band_cols, int32_t *units_out, int64_t *n_units_out) {
  cim::clear_error();
  if (n_tiles < 0 || nb < 1 || max_unit < 1 || band_cols < 1 || !n_units_out)
    return set_error(CIM_EINVAL, "bad arguments");
  if (n_tiles > 0 && (!rc || !units_out)) return set_error(CIM_EINVAL, "NULL arrays");
  if (n_tiles > INT32_MAX) return set_error(CIM_EINVAL, "n_tiles exceeds int32 range");
  int64_t nu = 0;
  int64_t t = 0;
  int64_t prev_band = -1;
  int32_t prev_R = -1;
  while (t < n_tiles) {
    const int32_t R = rc[2 * t];
    if (R < 0 || R >= nb) return set_error(CIM_EINVAL, "tile row out of range at index " + std::to_string(t));
    const int32_t C0 = rc[2 * t + 1];
    if (C0 < 0 || C0 >= nb) return set_error(CIM_EINVAL, "tile column out of range at index " + std::to_string(t));
    const int64_t band = C0 / band_cols;
    if (band < prev_band || (band == prev_band && R <= prev_R))
      return set_error(CIM_EINVAL, "tiles not sorted by (band, row) at index " + std::to_string(t));
    int64_t e = t;
    int32_t prevC = -1;
    while (e < n_tiles && rc[2 * e] == R && rc[2 * e + 1] / band_cols == band) {
      const int32_t C = rc[2 * e + 1];
      if (C < R) return set_error(CIM_EINVAL, "tile below the diagonal (C < R) at index " + std::to_string(e));
      if (C >= nb) return set_error(CIM_EINVAL, "tile column out of range at index " + std::to_string(e));
      if (C <= prevC) return set_error(CIM_EINVAL, "tiles not sorted/unique within row at index " + std::to_string(e));
      prevC = C;
      ++e;
    }
    for (int64_t s = t; s < e; s += max_unit) {
      const int64_t f = (s + max_unit < e) ? s + max_unit : e;
      units_out[4 * nu + 0] = R;
      units_out[4 * nu + 1] = static_cast<int32_t>(s);
      units_out[4 * nu + 2] = static_cast<int32_t>(f);
      units_out[4 * nu + 3] = 0;
      ++nu;
    }
    prev_band = band;
    prev_R = R;
    t = e;
  }
  *n_units_out = nu;
  return CIM_OK;
}

extern "C" int cim_plan_units(const int32_t *rc, int64_t n_tiles, int64_t nb, int32_t max_unit,
                              int32_t *units_out, int64_t *n_units_out) {
  return cim_plan_units_banded(rc, n_tiles, nb, max_unit, nb, units_out, n_units_out);
}

extern "C" int cim_partition_units(const int32_t *units, int64_t n_units, int32_t parts, int64_t *bounds) {
  cim::clear_error();
  if (parts < 1 || n_units < 0 || !bounds || (n_units > 0 && !units)) return set_error(CIM_EINVAL, "bad arguments");
  // prefix of tile counts; cut where the prefix crosses q·total/parts, but
  // never between units of the same block row (a row's acc_r flush is local).
  std::vector<int64_t> pre(n_units + 1, 0);
  for (int64_t u = 0; u < n_units; ++u) pre[u + 1] = pre[u] + (units[4 * u + 2] - units[4 * u + 1]);
  const int64_t total = pre[n_units];
  bounds[0] = 0;
  int64_t u = 0;
  for (int32_t q = 1; q < parts; ++q) {
    const double target = static_cast<double>(total) * q / parts;
    while (u < n_units && static_cast<double>(pre[u + 1]) <= target) ++u;
    // choose the closer of u and u+1 as the cut
    int64_t cut = u;
    if (u < n_units && (target - pre[u]) > (pre[u + 1] - target)) cut = u + 1;
    // snap to a block-row boundary (rows never straddle ranks)
    while (cut > 0 && cut < n_units && units[4 * cut] == units[4 * (cut - 1)]) ++cut;
    if (cut < bounds[q - 1]) cut = bounds[q - 1];
    bounds[q] = cut;
  }
  bounds[parts] = n_units;
  return CIM_OK;
}
