// common.hpp — internal types shared by the translation units behind include/slab_b200.h.
//
// Data layout in HBM (DESIGN.md has the long version):
//  * vectors: fp64, natural x-fastest order, n owned entries (+ ghost tail when decomposed);
//  * matrices: SELL-32 — rows grouped in slices of 32, a slice stores its entries slot-major
//    (slot k of all 32 rows contiguous: 256 B of values, 128 B of 32-bit column indices), slices
//    have individual widths. Padding slots carry column -1 and are skipped, so a row sum runs
//    over exactly the stored entries in ascending column order (operations.hpp:116-125);
//  * a level keeps its matrix twice: rows in natural order (SpMV / residual) and rows grouped by
//    colour (the Gauss-Seidel steps), each colour block padded to whole slices.
#pragma once

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/slab_b200.h"
#include "decomp.hpp"

namespace slabgpu {

	struct Error {
		int status;
		std::string message;
	};

	[[noreturn]] inline void fail( int status, const std::string & message ) {
		throw Error{ status, message };
	}

	inline void cuda_check( cudaError_t err, const char * what, const char * file, int line ) {
		if( err != cudaSuccess ) {
			fail( SLAB_ERR_CUDA, std::string( what ) + ": " + cudaGetErrorString( err ) + " (" + file + ":"
				+ std::to_string( line ) + ")" );
		}
	}
#define SLAB_CUDA( expr ) ::slabgpu::cuda_check( ( expr ), #expr, __FILE__, __LINE__ )

	// Host -> device copy ordered on `stream` and complete on return. (A plain cudaMemcpy from
	// pageable memory may return before the DMA has landed and is only ordered against the legacy
	// stream, which the library's non-blocking streams do not synchronise with.)
	inline void upload_sync( cudaStream_t stream, void * dst, const void * src, size_t bytes ) {
		if( bytes == 0 ) {
			return;
		}
		SLAB_CUDA( cudaMemcpyAsync( dst, src, bytes, cudaMemcpyHostToDevice, stream ) );
		SLAB_CUDA( cudaStreamSynchronize( stream ) );
	}

	extern uint64_t g_tuning_epoch;  // bumped by every slab_set_tuning: cached graphs are keyed by it
	extern size_t g_l2_persist_bytes;
	extern int g_dot_tile;            // exact dot: tile override (0 = automatic)
	extern int g_dot_cpb;             // exact dot: chunks per block override (0 = automatic)
	extern size_t g_l2_window_max;
	extern int g_l2_window;
	extern int64_t g_stream_rows;
	extern int g_stream_variant;
	extern std::atomic< uint64_t > g_launch_count; // kernels launched by this process (all contexts)
	extern int g_use_pdl; // chain kernels with programmatic dependent launch (default on)
	extern int g_use_packed;   // run products and colour steps from the dictionary-coded matrix copy when one exists
	extern int g_pack_build;   // build the dictionary-coded copy when a matrix is created
	extern int g_keep_plain;   // keep the plain arrays next to a coded copy without escaped rows (default 1)
	extern int g_packed_block; // threads per block of the packed kernels (tuning)
	extern int g_packed_batch;
	extern int g_packed_rows;
	extern int g_packed_rows_spmv;
	extern int64_t g_packed_multi_min_rows;
	extern int64_t g_cluster_rows;          // sweep_cluster.cu: largest colour of a level that takes the one-launch sweep (0 = off, default 384)
	extern int64_t g_packed_min_rows;
	extern int g_use_tile;            // tile.cu: shared-memory-staged kernels on stencil boxes (default 1)
	extern int64_t g_tile_min_rows;   // ... for colour pairs / products of at least this many rows
	extern int g_tile_ty, g_tile_cz, g_tile_ns; // tile shape overrides (0 = automatic)
	extern int g_use_planes;          // plane.cu: three-launch symmetric sweeps on regular box levels (default 1)
	extern int64_t g_plane_min_rows;  // ... for levels of at least this many rows
	extern int g_plane_ty, g_plane_cz, g_plane_ns, g_plane_rows; // shape overrides (0 = automatic)
	extern int g_use_spmv_planes;         // plane_spmv.cu: slab-staged products of regular box matrices (default 1)
	extern int64_t g_spmv_plane_min_rows; // ... for matrices of at least this many rows
	extern int g_spmv_plane_ty, g_spmv_plane_cz, g_spmv_plane_ns; // shape overrides (0 = automatic)
	extern int g_plane_unit;          // plane.cu: additions of -e where every off-diagonal value is -1.0 (default 1)
	extern int g_plane_autotune;      // plane.cu: measure proposed tile shapes at level creation (default 1)
	extern int g_lazy_x;              // cg.cu: fixed-iteration solves take cg.hpp:128 one iteration late, on a side stream under the coarse levels of the next V-cycle (default 1)
	extern int g_lazy_x_prio;         // ... the iteration graph runs its nodes with the priorities of the streams they were captured on (default 1)
	extern int g_iter_batch;          // cg.cu: CG iterations per graph launch in fixed-iteration solves (the largest divisor of the count up to this; default 50)
	extern int g_inline_record;       // cg.cu: the history entry and the iteration count ride on the p and r updates (default 1)
	extern int g_lazy_x_blocks;       // ... blocks per SM of that pass (default 1)
	extern int g_side_rr;             // cg.cu: exact-dot mode, r'r on a side stream beside the next V-cycle (default 1)
	extern int g_fuse_rz;             // cg.cu: r'z on the last plane phases of the V-cycle in tree-dot mode (default 1)
	extern int g_plane_pad_lines;     // plane.cu: pad lines to a divisor of 32 threads (0 never, 1 up to 35 % idle, 2 always)
	extern int g_plane_warp_sync;     // plane.cu: warp instead of block barriers between the x-parity colours of a line (default 1)
	// launches a thread has counted so far: a stream capture counts its enqueues here and takes them back from
	// the process-wide counter afterwards (they run when the graph is replayed, and are counted then)
	inline uint64_t & thread_launches() {
		thread_local uint64_t count = 0;
		return count;
	}
	inline void count_launch( uint64_t k = 1 ) {
		g_launch_count += k;
		thread_launches() += k;
	}

	constexpr int kSlice = 32;            // rows per SELL slice = one warp
	constexpr uint64_t kDotChunk = 4096;  // parallel.hpp:70

	// device scalar slots used by the CG driver (doubles in ctx->d_scalars)
	// S_RHO and S_RR are neighbours: on a communicator r'z of an iteration and r'r of the one before travel in ONE
	// allreduce of two doubles (cg.cu)
	enum Scalar { S_RHO = 0, S_RR, S_RHO_PREV, S_PQ, S_TMP, S_BB, S_ALPHA, S_COUNT = 16 };

	// Dictionary-coded companion of a SELL matrix (packed.cu). Every stored entry is replaced by one
	// byte: the index of its (column - row, value) pair in a dictionary of at most 254 pairs found in
	// the matrix itself. Code 0 is padding; a row whose first code is 255 has an entry outside the
	// dictionary and is read from the plain SELL arrays instead. A row occupies `chunks` 16-byte words,
	// slice-interleaved like the SELL arrays: word j of lane l of slice s at [(s*chunks + j)*32 + l].
	// The last byte of a row's words holds the code of its diagonal entry (0 = none).
	struct alignas( 16 ) DictEntry {
		double val;
		int32_t delta;
		int32_t unused;
	};
	struct Packed {
		int max_width = 0;         // widest row (stored entries)
		int ncodes = 0;            // width class the kernels are instantiated for (>= max_width)
		int chunks = 0;            // 16-byte words stored per row = (ncodes + 16) / 16
		uint4 * codes = nullptr;   // device
		DictEntry * dict = nullptr; // device, 256 entries, entry 0 = {0.0, 0} (read by the encoder)
		DictEntry * h_dict = nullptr; // host copy: the kernels take the dictionary as a launch parameter
		int dict_size = 0;         // entries in use, including entry 0
		int64_t escaped_rows = 0;  // rows that fall back to the plain arrays
		int stride = 0;            // slices between rows that mostly repeat their codes (0 = no such distance)
		void release();
		bool usable() const {
			return codes != nullptr;
		}
	};

	struct Sell {
		int64_t nrows = 0;     // logical rows (positions), multiple of kSlice not required
		int64_t nslices = 0;
		int64_t entries = 0;   // stored slots incl. padding
		int max_width = 0;     // widest slice
		Packed packed;         // optional, see sell_pack
		int64_t * slice_off = nullptr; // device, nslices+1, in entries
		double * vals = nullptr;       // device
		int32_t * cols = nullptr;      // device, -1 = padding
		void release();
		bool plain_dropped() const { // the plain arrays were freed (g_keep_plain == 0): only the coded copy is left
			return vals == nullptr && packed.usable();
		}
		uint64_t bytes() const {
			return ( plain_dropped() ? 0u : static_cast< uint64_t >( entries ) * 12u ) + static_cast< uint64_t >( nslices + 1 ) * 8u;
		}
		uint64_t packed_bytes() const {
			return packed.usable() ? static_cast< uint64_t >( nslices ) * packed.chunks * kSlice * 16u + 256u * 16u : 0u;
		}
	};

	// Bitmap-coded companion of a coded matrix whose rows live on a 3D box (tile.cu). When every (column - row,
	// value) pair of the dictionary is one of the 27 offsets dx + lx*(dy + ly*dz), |d| <= 1, with ONE value per
	// offset, a row is the subset of those 27 pairs it stores: a 32-bit mask (bit 9*(dz+1) + 3*(dy+1) + (dx+1)),
	// built from the row's codes and checked entry by entry when the matrix is created. Ascending bit order is
	// ascending column order, so the ordered row sum of operations.hpp:116-125 walks the set bits. 4 bytes per
	// row instead of 32; the kernels that read it stage the vector through shared memory with bulk-async copies.
	struct BoxTile {
		uint32_t * masks = nullptr; // device, one per row position (0 on padding positions)
		double vals[ 27 ] = { 0.0 };  // the value of each offset (0.0: offset not in the dictionary)
		int lx = 0, ly = 0, lz = 0;
		// every row stores exactly the offsets that stay inside the box, all 27 values are finite: the kernels of
		// plane.cu need no masks then (zero-padded slabs stand in for the absent neighbours)
		bool regular = false;
		// plane.cu: tile shape (ty, cz, ns) of phases A, B, C as measured when the level was built (0: not measured)
		int tuned[ 5 ][ 3 ] = { { 0 } };
		void release();
		bool usable() const {
			return masks != nullptr;
		}
	};

	struct CgWorkspace;
	struct DistState; // dist.cu: process grid + NCCL communicator of a context
	struct HaloPlan;  // dist.cu: per-level send lists / ghost layout

} // namespace slabgpu

namespace slabgpu {
	// a device-time interval whose length is added (or subtracted) to a LevelStats counter once resolved
	struct TimedSpan {
		cudaEvent_t begin, end;
		uint64_t * target;
		int sign;
	};
} // namespace slabgpu

struct slab_ctx_s {
	slabgpu::DistState * dist = nullptr; // null: single-process context
	// LevelStats timing (problem.hpp:204-209): when on, V-cycles run launch by launch (no graphs, no
	// fusion across the reference's categories) with CUDA events around the sections the reference
	// wraps with its monotonic clock; intervals are resolved lazily when the stats are read
	int profiling = 0;
	std::vector< slabgpu::TimedSpan > spans;
	std::vector< cudaEvent_t > event_pool;
	int device = 0;
	cudaStream_t stream = nullptr;
	int sm_count = 0;
	int cc_major = 0, cc_minor = 0;
	uint64_t hbm_bytes = 0;
	int dot_mode = SLAB_DOT_EXACT;
	int use_graphs = 1;
	int fused_transfers = 1;
	double * d_scalars = nullptr;   // S_COUNT doubles
	double * d_partials = nullptr;  // reduction scratch
	uint64_t partials_cap = 0;
	uint64_t scratch_gen = 0;       // bumped whenever d_partials moves: part of every cached graph's key
	unsigned int * d_counter = nullptr; // "last block done" tickets (zeroed, self-resetting); [1] belongs to the side stream
	// exact-dot solves: r'r (needed for the history only) runs on a side stream beside the next V-cycle (cg.cu)
	cudaStream_t side_stream = nullptr;
	cudaEvent_t side_fork = nullptr, side_join = nullptr;
	// lazy x (cg.cu): the x update of the previous iteration on its own low-priority stream, forked by the V-cycle after
	// the finest level's pre-smoother (level.cu takes `after_presmooth` once)
	cudaStream_t lazy_stream = nullptr;
	cudaEvent_t lazy_fork = nullptr, lazy_join = nullptr;
	std::function< void() > after_presmooth;
	double * d_partials_side = nullptr;
	uint64_t partials_side_cap = 0;
	double * h_pinned = nullptr;    // pinned staging for scalar read-back
	uint64_t h_pinned_cap = 0;
	cudaEvent_t timer_start = nullptr, timer_stop = nullptr; // slab_ctx_timer_* (caller-owned interval)
	cudaEvent_t solve_start = nullptr, solve_stop = nullptr; // cg_solve's own interval (slab_cg_result::solve_ms)
};

struct slab_vec_s {
	slab_ctx_s * ctx = nullptr;
	uint64_t n = 0;      // owned entries
	uint64_t n_alloc = 0; // owned + ghost tail
	double * d = nullptr;
	~slab_vec_s() {
		if( d ) {
			cudaFree( d );
		}
	}
};

struct slab_mat_s {
	slab_ctx_s * ctx = nullptr;
	uint64_t nrows = 0, ncols = 0, nnz = 0;
	slabgpu::Sell sell;             // natural row order
	slabgpu::HaloPlan * plan = nullptr; // borrowed from the level: columns >= ncols are ghost slots
	slabgpu::BoxTile tile;          // optional (stencil boxes on one process): natural-order rows as masks, tile.cu
	std::unique_ptr< slab_mat_s > transposed; // built lazily for SLAB_DESC_TRANSPOSE
	// host CSR kept when the matrix came from slab_mat_create_csr (small, test-sized inputs)
	std::vector< uint64_t > h_row_offsets, h_cols;
	std::vector< double > h_vals;
	bool has_host_csr = false;
	~slab_mat_s() {
		sell.release();
	}
};

struct slab_mask_s {
	slab_ctx_s * ctx = nullptr;
	uint64_t universe = 0, count = 0;
	int32_t * d_members = nullptr;
	~slab_mask_s() {
		if( d_members ) {
			cudaFree( d_members );
		}
	}
};

struct slab_level_s {
	slab_ctx_s * ctx = nullptr;
	uint64_t dims[ 3 ] = { 0, 0, 0 };
	uint64_t n = 0, nnz = 0;
	bool is_stencil = false;
	std::unique_ptr< slab_mat_s > A;       // natural-order SELL
	slabgpu::Sell colorA;                  // colour-major SELL (positions)
	slabgpu::BoxTile tile;                 // optional: colour-major rows as masks (tile.cu)
	int32_t * d_rows = nullptr;            // position -> natural row, -1 on padding
	slabgpu::Decomp decomp{};              // owned box of this rank on this level (whole grid when not distributed)
	slabgpu::HaloPlan * plan = nullptr;    // owned; null on single-process contexts and general levels
	uint64_t num_colors = 0;
	std::vector< int64_t > color_pos;      // first position of colour k (multiple of 32); size num_colors+1
	std::vector< uint64_t > color_size;    // members per colour
	std::vector< uint64_t > color_nnz;     // stored nonzeros per colour (problem.hpp:237-245)
	std::unique_ptr< slab_vec_s > a_diag;
	std::unique_ptr< slab_mat_s > R;       // restriction (n_c x n), null at the coarsest
	std::unique_ptr< slab_level_s > coarser;
	std::unique_ptr< slab_vec_s > s, f, r_c, z_c; // scratch (problem.hpp:228-231)
	std::unique_ptr< slab_vec_s > zs;             // plane.cu: the out-of-place partner of the smoothed vector
	bool planes_ok = false;                       // the level can run the plane phases of plane.cu
	slab_level_stats stats{};
	// V-cycle graph cache (keyed by the vectors it was captured with)
	cudaGraphExec_t vcycle_exec = nullptr;
	double * vcycle_z = nullptr;
	double * vcycle_r = nullptr;
	uint64_t vcycle_sweeps = 0;
	int vcycle_fused = -1;
	uint64_t vcycle_epoch = ~uint64_t( 0 );
	uint64_t vcycle_scratch = ~uint64_t( 0 );
	uint64_t vcycle_launches = 0;
	// CG workspace of the hierarchy head: r, z, p, q, device history, iteration graph
	std::unique_ptr< slabgpu::CgWorkspace > cg;
	~slab_level_s();
};

namespace slabgpu {

	struct CgWorkspace {
		std::unique_ptr< slab_vec_s > r, z, p, q;
		std::unique_ptr< slab_vec_s > host_b, host_x; // device staging of slab_cg_solve_host
		double * d_hist_rr = nullptr;
		double * d_hist_pq = nullptr;
		unsigned int * d_iter = nullptr;
		uint64_t hist_cap = 0;
		cudaGraphExec_t iter_exec = nullptr;
		double * key_x = nullptr;
		uint64_t key_sweeps = 0;
		int key_precond = -1, key_dot = -1, key_fused = -1;
		uint64_t key_epoch = ~uint64_t( 0 );
		uint64_t key_scratch = ~uint64_t( 0 );
		int key_deferred = -1;
		uint64_t key_batch = 0;
		uint64_t iter_launches = 0;
		~CgWorkspace();
	};

	// ---- containers.cu
	slab_vec_s * vec_new( slab_ctx_s * ctx, uint64_t n, double value );
	void vec_free( slab_vec_s * v );
	void ensure_partials( slab_ctx_s * ctx, uint64_t count );
	void ensure_pinned( slab_ctx_s * ctx, uint64_t doubles );
	double read_scalar( slab_ctx_s * ctx, int slot ); // syncs the stream
	slab_mat_s * mat_from_csr( slab_ctx_s * ctx, uint64_t nrows, uint64_t ncols, const uint64_t * ro,
		const uint64_t * co, const double * va, bool validate );
	slab_mat_s * mat_stencil27( slab_ctx_s * ctx, uint64_t nx, uint64_t ny, uint64_t nz );
	slab_mat_s * mat_stencil27_box( slab_ctx_s * ctx, const Decomp & D ); // rows of the owned box, ghost columns
	slab_mat_s * mat_restriction( slab_ctx_s * ctx, uint64_t nx, uint64_t ny, uint64_t nz );
	void mat_download_csr( slab_mat_s * A, uint64_t * ro, uint64_t * co, double * va );
	slab_mat_s * mat_transposed( slab_mat_s * A );
	// SELL over an arbitrary list of rows of a host CSR (row -1 = empty padding row)
	Sell sell_from_csr_rows( slab_ctx_s * ctx, const std::vector< int64_t > & rows, const uint64_t * ro,
		const uint64_t * co, const double * va );
	// SELL of the 27-point stencil over an arbitrary device row list (d_rows == nullptr: natural order)
	Sell sell_stencil27( slab_ctx_s * ctx, const Decomp & D, const int32_t * d_rows, int64_t npos );
	// packed.cu: build S.packed from the entries of S (d_rows: position -> row, nullptr = identity);
	// leaves S.packed unusable when the matrix does not compress (rows wider than 64 entries, or
	// too many rows with entries outside a 254-pair dictionary)
	// owned_cols: columns from this index on are ghost slots (never offered to the dictionary); < 0: none
	void sell_pack( slab_ctx_s * ctx, Sell & S, const int32_t * d_rows, int64_t owned_cols = -1 );
	Decomp single_domain( uint64_t nx, uint64_t ny, uint64_t nz );
	// tile.cu: build T from the coded copy of S (rows: position -> natural row, nullptr = identity) on the box D;
	// leaves T unusable when the matrix is not a subset-of-27-offsets matrix on that box
	void box_tile_build( slab_ctx_s * ctx, const Sell & S, const int32_t * d_rows, const Decomp & D, BoxTile & T );
	// coloring.cu: greedy_color (coloring.hpp:114-158) as a device wavefront; color[i] per row
	void greedy_color_device( slab_ctx_s * ctx, uint64_t n, const uint64_t * ro, const uint64_t * co, std::vector< int32_t > & color, uint64_t & num_colors );
	// is d_rows the parity lattice of the box (colour c = px + 2 py + 4 pz, members x-fastest)? The colour-pair
	// kernel computes row positions from coordinates instead of reading the list.
	bool box_tile_lattice_ok( slab_ctx_s * ctx, const int32_t * d_rows, const std::vector< int64_t > & color_pos, const Decomp & D );

	// ---- dist.cu (3D domain decomposition, halo exchange, allreduce)
	Decomp level_decomp( const slab_ctx_s * ctx, uint64_t lx, uint64_t ly, uint64_t lz ); // owned box of this rank
	uint64_t ghost_capacity( const slab_ctx_s * ctx );
	HaloPlan * halo_plan_create( slab_ctx_s * ctx, const Decomp & D );
	void halo_plan_destroy( HaloPlan * plan );
	// bring the ghost copies of v up to date: colour < 0 exchanges every colour. No-op on
	// single-process contexts and in manual-exchange mode (no communicator attached).
	void halo_exchange( slab_level_s * L, slab_vec_s * v, int color );
	void halo_exchange_plan( slab_ctx_s * ctx, HaloPlan * plan, slab_vec_s * v, int color, cudaStream_t stream = nullptr );
	// boundary rows of every colour as colour-major positions (level.cu computes them, the plan owns them)
	void halo_plan_set_boundary( slab_ctx_s * ctx, HaloPlan * plan, const std::vector< std::vector< int32_t > > & per_color,
		int64_t npos );
	bool halo_overlap_active( const slab_ctx_s * ctx, const HaloPlan * plan ); // split colour steps into boundary + interior?
	bool halo_has_comm( const slab_ctx_s * ctx );
	void halo_fork( slab_ctx_s * ctx );  // comm stream waits for what the main stream has enqueued so far
	void halo_join( slab_ctx_s * ctx );  // main stream waits for what the comm stream has enqueued so far
	cudaStream_t halo_comm_stream( slab_ctx_s * ctx );
	const int32_t * halo_boundary_positions( const HaloPlan * plan, int color, int64_t * count );
	const uint8_t * halo_boundary_flags( const HaloPlan * plan );
	extern int g_halo_overlap;
	void allreduce_slot( slab_ctx_s * ctx, int slot ); // sum d_scalars[slot] over ranks, in place
	void allreduce_slots( slab_ctx_s * ctx, int slot, int count ); // ... d_scalars[slot .. slot + count)
	void dist_destroy( slab_ctx_s * ctx );

	// ---- level.cu
	slab_level_s * hierarchy_create( slab_ctx_s * ctx, uint64_t nx, uint64_t ny, uint64_t nz, uint64_t levels );
	slab_level_s * level_from_csr( slab_ctx_s * ctx, uint64_t n, const uint64_t * ro, const uint64_t * co,
		const double * va );
	void rbgs_color_step( slab_level_s * L, uint64_t k, slab_vec_s * z, slab_vec_s * r );
	void rbgs_color_step_twice( slab_level_s * L, uint64_t k, slab_vec_s * z, slab_vec_s * r );
	void rbgs_forward( slab_level_s * L, slab_vec_s * z, slab_vec_s * r );
	void rbgs_backward( slab_level_s * L, slab_vec_s * z, slab_vec_s * r );
	void rbgs_symmetric( slab_level_s * L, slab_vec_s * z, slab_vec_s * r, uint64_t sweeps );
	void restrict_vector( slab_level_s * L, slab_vec_s * v_fine, slab_vec_s * out );
	void refine_and_add( slab_level_s * L, slab_vec_s * z, slab_vec_s * z_c );
	void mg_vcycle( slab_level_s * L, slab_vec_s * z, slab_vec_s * r, uint64_t sweeps );
	void mg_vcycle_enqueue( slab_level_s * L, slab_vec_s * z, slab_vec_s * r, uint64_t sweeps, bool count_stats, bool zero_guess = false,
		bool fuse_rz = false );
	uint64_t mg_vcycle_rz_partials( const slab_level_s * L ); // partials the fused r'z leaves in ctx->d_partials
	// does the V-cycle rooted at L take the "z is zero" hint on its first phase (so that the caller need not zero z)?
	bool mg_vcycle_accepts_zero_guess( const slab_level_s * L );
	// everything mg_vcycle_enqueue needs that may allocate or copy (phase lists of the persistent kernel,
	// lazily built transposes): must run before stream capture begins
	void mg_vcycle_prepare( slab_level_s * L, slab_vec_s * z, slab_vec_s * r, uint64_t sweeps );
	void spans_resolve( slab_ctx_s * ctx ); // synchronises; adds every pending interval to its counter
	void spans_discard( slab_ctx_s * ctx );

	// ---- ops (kernels.cu)
	void op_set_all( slab_vec_s * v, double value );
	void op_waxpby( slab_vec_s * w, double alpha, slab_vec_s * x, double beta, slab_vec_s * y );
	// result -> ctx->d_scalars[slot]; reduce = false leaves this rank's part there (the caller combines allreduces)
	void op_dot_to_slot( slab_vec_s * x, slab_vec_s * y, int slot, bool reduce = true );
	double op_dot( slab_vec_s * x, slab_vec_s * y );
	void op_mxv( slab_vec_s * y, slab_mask_s * mask, slab_mat_s * A, slab_vec_s * x, unsigned desc );

	// ---- cg.cu
	void cg_solve( slab_level_s * H, slab_vec_s * b, slab_vec_s * x0, const slab_cg_config * cfg, slab_vec_s * x,
		double * history, slab_cg_result * result );
	void cg_solve_host( slab_level_s * H, const double * b, const double * x0, const slab_cg_config * cfg, double * x,
		double * history, slab_cg_result * result );
	double residual_norm( slab_mat_s * A, slab_vec_s * x, slab_vec_s * b );

} // namespace slabgpu
