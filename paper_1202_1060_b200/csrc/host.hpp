// host.hpp -- host-side code graphs and CN-group schedules.
//
// This is the single source of truth for H and the grouping: the B200 kernels
// and the CPU oracle both consume the arrays built here, so construction and
// grouping are bit-exact by construction.
//
// Reference interfaces mirrored:
//   CodeData      <- ldpc::TannerGraph            tanner.hpp:21-37
//   build_code    <- ldpc::build_from_check_lists tanner.hpp:79-114
//   regular_rows  <- ldpc::random_regular_graph   tanner.hpp:356-393
//   parse_alist / serialize_alist                 tanner.hpp:163-317
//   ScheduleData  <- ldpc::GroupSchedule          schedule.hpp:32-40
//   random_groups <- detail::generate_groups      schedule.hpp:54-115
//   iteration_budget / measure_cocsg              schedule.hpp:175-210
#pragma once
#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace ldpcb {

using Rows = std::vector<std::vector<int>>;

// CN-major edge numbering: edge (check m, slot k) = row_off[m] + k. The VN
// view lists CN ids ascending with the matching edge ids.
struct CodeData {
  int n = 0, m = 0, E = 0;
  int max_cdeg = 0, max_vdeg = 0;
  std::vector<int32_t> row_off, cols;
  std::vector<int32_t> var_off, var_cns, var_edges;
};

// Alist errors carry the reference's kind enumeration and 1-based line.
enum class AlistKind {
  malformed_header = 0,
  bad_token,
  degree_error,
  length_mismatch,
  index_out_of_range,
  duplicate_entry,
  edge_count_mismatch,
  transpose_mismatch,
  trailing_content,
  truncated,
};

struct AlistFailure : std::runtime_error {
  AlistKind kind;
  int line;
  AlistFailure(AlistKind k, int l, const std::string& what)
      : std::runtime_error("alist parse error at line " + std::to_string(l) + ": " + what), kind(k), line(l) {}
};

CodeData build_code(int n_vars, const Rows& rows);
Rows rows_of(const CodeData& c);

Rows regular_rows(int n_vars, int dv, int dc, uint64_t seed);
// Edge swaps until no two CNs share two VNs (girth >= 6); degrees preserved.
void break_4cycles(int n_vars, Rows& rows, uint64_t seed);
// Quasi-cyclic base-matrix expansion (BASELINE config 3).
Rows qc_rows(int base_rows, int base_cols, int z, double p_empty, int min_col_degree, uint64_t seed);
// Socket-matched irregular VN / regular CN ensemble (BASELINE config 4).
Rows irregular_rows(int n_vars, const std::vector<int>& degrees, const std::vector<int>& counts, int dc,
                    uint64_t seed);
int64_t count_4cycles(const CodeData& c);

CodeData parse_alist(std::string_view text);
std::string serialize_alist(const CodeData& c);

enum class Kind { flooding = 0, disjoint = 1, nondisjoint = 2 };

struct ScheduleData {
  Kind kind = Kind::flooding;
  int G = 1;
  double overlap = 0.0;
  int group_size = 0;
  uint64_t seed = 0;
  std::vector<int32_t> grp_off, grp_cns;      // groups in processing order
  std::vector<int32_t> touch_off, touch_vns;  // sorted unique VNs per group
  int64_t edge_updates_per_iter = 0;          // sum of CN degrees over group slots
  int64_t touched_per_iter = 0;               // sum of touched-set sizes
  int max_group = 0, max_touched = 0;
  // Per-frame random grouping (the reference harness, sim.hpp:113-117):
  // frame f uses generate_groups(M, G, r, Rng(mix_seed(mix_seed(schedule_seed,
  // f), it))) in iteration it = 1, and again for every it > 1 when regroup
  // is set (decoder.hpp:153-156). grp_off / grp_cns then hold frame 0's
  // iteration-1 groups; the offsets are the same for every frame.
  bool per_frame = false;
  bool regroup = false;
  int nominal = 0, k_overlap = 0;
};

// Compact per-group records read by the resident kernel (one vectorised,
// frame-broadcast load per CN or VN item). c2v lives in "slots": for
// check-regular codes slot(m, k) = m * slot_stride + k with an ODD stride, so
// the consecutive CNs of a window hit distinct shared-memory banks; otherwise
// CN r owns (deg r | 1) consecutive slots (odd again, so consecutive CNs of one
// degree hit distinct banks). The last slot is always zero (pads VN records).
//   CN record  [slot of edge 0, single-touch mask, pos(v_0) .. pos(v_{d-1}), -1 ...]  cs ints
//   VN record  [pos(v), slot_0 .. slot_{d-1} (ascending CN), zero slot ...] 4*vs4 ints
// Bit k of the mask is set when v_k has no other CN in the group: the CN
// thread then updates that VN's posterior in place; VNs shared by two or more
// CNs of the group ("fix" records) are re-summed after the CN phase.
// A CN listed twice in one group is kept once (its second update would read
// the same pre-group messages and write the same values).
struct KernelTables {
  int cs = 0, vs4 = 0;
  int slot_stride = 0;     // 0: irregular rows, odd per-CN slot counts
  int n_slots = 0;         // including the zero slot
  bool recompute = false;  // some CN updates a posterior in place
  std::vector<int32_t> cn_off, cn_rec;    // per group
  std::vector<int32_t> fix_off, fix_rec;  // per group: VNs shared by >= 2 CNs
  // the same fix-up records with 16-bit fields (codes with < 2^16 slots and
  // VN records longer than one row): [pos, slot_0 .. slot_{d-1}, zero ...] as
  // uint16, eight per 16-byte row, vs16 rows per record (0: not built)
  std::vector<int32_t> fix_rec16;
  std::vector<int32_t> tot_rec16;  // tot_vn_rec with 16-bit fields (vs16 > 0)
  int vs16 = 0;
  std::vector<int32_t> all_vn_rec;        // every VN, record p = the VN at position p (decoder.hpp:162-165)
  std::vector<int32_t> tot_vn_rec;        // the same records in bank-coloured order (exact totals)
  std::vector<int32_t> all_rec;           // every CN in index order (syndrome)
  std::vector<int32_t> edge_slot;         // CN-major edge id -> slot
  // VN v lives at position vn_pos[v] of the kernels' per-VN arrays (P, L):
  // every record holds positions, not VN ids (bank colouring relabels VNs)
  std::vector<int32_t> vn_pos;
  int max_cn_items = 0, max_fix_items = 0;
  // Fresh frames (HBM-streamed frame queue, stream.cu): a lane refilled with a
  // new frame at an iteration boundary keeps the previous frame's c2v and
  // posteriors; during its first iteration the kernels read the values that
  // zero c2v and P = L would give, from static per-record bits:
  //   cn_fresh[i]  (per cn_rec record) bit 31: first processing of the CN in
  //                iteration order (its old c2v counts as 0); bit k: the VN at
  //                position k is touched by no earlier group (read L, not P)
  //   fix_fresh[i] (per fix_rec record) bit j: slot field j (0 = first slot)
  //                belongs to a CN processed in this group or an earlier one
  // covers: every CN is in some group and every VN is touched (the first
  // iteration then leaves no stale value behind).
  std::vector<uint32_t> cn_fresh, fix_fresh;
  bool covers = false;
};

// cs = CN record stride in ints (>= 2 + max CN degree, multiple of 4)
KernelTables kernel_tables(const CodeData& c, const ScheduleData& s, int cs, bool regular_rows);


// Tables of the direct (posterior-free) resident kernel (direct.cu) for codes
// whose VNs all have degree 3 and whose CNs all have degree 6. The state of
// the fv (2 or 4) frames a CTA decodes is one array of cells of fv floats (one
// per frame): a cell per edge and an L cell per VN (clamped channel LLR).
// Every VN has one "holder" edge, chosen so that every CN holds exactly two
// (a perfect matching): the holder's cell stores c2v + L, the other two
// edges' cells the plain c2v. A CN item then forms (var_update)
//   holder edge   v2c = (c2v_x + c2v_y) + L        three reads
//   other edges   v2c = (c2v_h + L) + c2v_o        two reads (the holder cell and the third edge's)
// i.e. 14 reads and 6 writes per CN, and no posterior array, in-place update
// or fix-up pass exist. Every field is a 16-bit byte offset into the cell
// array (cells * 4 fv <= 65536):
//   CN record  12 ints (10 used): positions 0, 1 = the CN's holder edges as
//              own | r0 << 16, r1 | L << 16; then positions 2..5 as the
//              16-bit triples own, r0, r1 packed two per word
//   VN record   2 ints, indexed by VN position: holder | second << 16, third
//              (hard decisions: total = (holder + second) + third)
//   vn_hold     per VN id: its holder cell (frame refill writes L there)
//   all_cn      4 ints per CN: the six VN positions as 16-bit fields (syndrome)
//   edge_rec    2 ints per CN-major edge id: own | (holder ? L : 0xffff) << 16, r0 | r1 << 16 (state dumps)
// Cell ids, record positions and read orders are bank-coloured
// (host_direct.cpp): the cells a wavefront touches in one instruction fall in
// distinct banks where possible.
struct DirectTables {
  bool ok = false;
  int fv = 2;        // frames per cell (2: 8-byte cells, 4: 16-byte cells)
  int cells = 0;     // cells, multiple of 16
  int l_base = 0;    // L cell of position p = l_base + p
  int buf_cells = 0; // flooding (one group of more CNs than a CTA has threads): the edge cells exist twice,
                     // buffer 1 = buffer 0 + buf_cells; an iteration reads one and writes the other. 0: one buffer
  int max_items = 0;
  double wavefronts = 0.0;  // shared-memory wavefronts per half-warp access after bank colouring (1 = conflict-free)
  std::vector<int32_t> cn_off, cn_rec, vn_rec, vn_hold, all_cn, edge_rec, vn_pos;
};
DirectTables direct_tables(const CodeData& c, const ScheduleData& s, int fv);

ScheduleData schedule_from_groups(const CodeData& c, Kind kind, const Rows& groups);
ScheduleData flooding_schedule(const CodeData& c);
ScheduleData reference_random_schedule(const CodeData& c, Kind kind, int G, double overlap, uint64_t seed);
ScheduleData window_schedule(const CodeData& c, Kind kind, int G, int window, int stride);
ScheduleData per_frame_schedule(const CodeData& c, Kind kind, int G, double overlap, uint64_t schedule_seed,
                                bool regroup);
Rows random_groups(int M, int G, double overlap, uint64_t stream_seed_value);
int iteration_budget(const ScheduleData& s, int n_checks, int i_max);
std::vector<int> measure_cocsg(const CodeData& c, const ScheduleData& s);

// Jump-ahead of the channel stream (host_rng.cpp): coefficients of
// x^draws mod p(x), p the characteristic polynomial of xoshiro256, and their
// application to a stream state (the published jump() loop).
struct Stream;
std::array<uint64_t, 4> stream_jump_poly(uint64_t draws);
void stream_jump(Stream& st, const std::array<uint64_t, 4>& poly);

}  // namespace ldpcb
